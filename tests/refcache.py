"""On-disk cache of ORACLE outputs for the GPU parity tests.

Every stored array is written by ``tests/golden/make_oracle_refs.py``, which
calls only ``oracle/`` (and the seeded generators in ``synth/``) — never the
CUDA path (task rule ③: "a stored value is ... written by a committed script
that calls only oracle/").  The GPU box then compares against these instead of
re-running the slow fp64 oracle in every round-end test run.  A missing entry
is computed on the spot (same function), so the cache is an optimisation only.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_refs")


def key_path(key: dict) -> str:
    h = hashlib.sha1(json.dumps(key, sort_keys=True, default=str).encode()).hexdigest()[:20]
    return os.path.join(DIR, h + ".npy")


def cached(key: dict, compute):
    """Return the oracle result for `key`, from disk if present.  With
    STADI_WRITE_REFS=1 a computed result is stored (make_oracle_refs.py)."""
    p = key_path(key)
    if os.path.exists(p):
        _KEYS[os.path.basename(p)] = key
        return np.load(p)
    out = compute()
    if os.environ.get("STADI_WRITE_REFS") == "1":
        os.makedirs(DIR, exist_ok=True)
        np.save(p, np.asarray(out, dtype=np.float64))
        _KEYS[os.path.basename(p)] = key
        with open(os.path.join(DIR, "index.jsonl"), "a") as f:
            f.write(json.dumps({"file": os.path.basename(p), "key": key}, sort_keys=True, default=str) + "\n")
    return out


_KEYS: dict = {}


def rewrite_index():
    """index.jsonl = one line per .npy present whose key this process saw
    (make_oracle_refs.py visits every case); files no case refers to are removed."""
    lines = []
    for f in sorted(os.listdir(DIR)):
        if not f.endswith(".npy"):
            continue
        if f not in _KEYS:
            os.remove(os.path.join(DIR, f))
            continue
        lines.append(json.dumps({"file": f, "key": _KEYS[f]}, sort_keys=True, default=str))
    with open(os.path.join(DIR, "index.jsonl"), "w") as f:
        f.write("\n".join(lines) + "\n")
