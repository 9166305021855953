"""STADI oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the STADI hot
path computes (arXiv 2509.04719, /root/reference/PAPER.md), written from the
paper in its own order and notation, in float64 numpy (exact integers /
``fractions`` for the planner).  It exists to check the CUDA path.

Rules (task brief ③):
* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import or execute it.  The
  product path (``paper_2509_04719_b200``) never imports it and shares no code
  with it; the only shared module is ``synth`` (seeded inputs, no arithmetic).
* Every function cites the passage it follows (PAPER.md line numbers, section,
  equation, algorithm line) or the SURVEY.md §8(c) reading (R#) where the paper
  is silent.

Modules
-------
planner   Eq. 4 step allocator + Eq. 5 patch sizer        — pinned
schedule  per-rank step table, Alg. 1 lines 8-24, Thm 2 grid (O2)   — pinned
diffusion noise schedule + Eq. 3 DDIM/DPM-Solver-1 update (O3)      — pinned
dit       DiT-family eps_theta, full and band (patch) forward (O4/O5) — pinned
stadi     Algorithm 1 end to end, all ranks simulated in one process (O6)

unet      U-Net-family eps_theta, band forward with exchange sites     — pinned

Parity status: the stale-activation protocol (which version each site
reads) has no worked example in the paper; beyond the reductions pinned in
tests/test_oracle_model.py and tests/test_oracle_unet.py (fresh exchange ==
unpatched, time-invariant activations make staleness exact) it is "parity
unpinned".
"""
from . import planner, schedule, diffusion, dit, stadi, unet  # noqa: F401
