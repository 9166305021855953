"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no planner, no schedule, no
model, no sampler).  It only describes the workloads (BASELINE.json configs
C1..C5, SURVEY.md §8(d) "Common inputs") and draws their inputs:

* ``configs``  — the model/run presets (shapes, step counts, guidance, seeds).
* ``gen``      — seeded numpy generators: random-init weights in manifest order
                 (SURVEY §8(c) R22), initial noise x_T (R21/§8(d)), conditioning
                 (class labels / synthetic text embeddings, R21), and the bf16
                 round-to-nearest-even input transform used by bf16 parity runs.

Both ``oracle/`` and ``paper_2509_04719_b200`` import it; neither imports the
other.
"""
from . import configs, gen  # noqa: F401
