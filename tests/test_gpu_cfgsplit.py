"""R33 CFG batch split on the GPU: each GPU (local-mode rank, IPC process or virtual
GPU) computes one CFG branch (B = 1) of its pair's band, K/V travel only within a
branch, the pair swaps its eps rows every step.  Checked against the fp64 oracle's
unsplit run of the pair plan (oracle/stadi.py run_cfg_split == run(pair_plan) is
pinned on the CPU), and multi-process / virtual-GPU runs against local mode bit for
bit."""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

from oracle import planner as OP
from oracle import stadi as OR
from synth import configs, gen
import refcache

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-2
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "helpers", "ipc_worker.py")
CASES = [  # id, name, kwargs, speeds, m_base, m_warmup
    ("c2_4gpu_tier2", "dit_xl2", dict(depth=2), [65536, 39322, 60000, 30000], 50, 4),
    ("c5red_2gpu", "pixart_alpha", dict(depth=2, latent_h=32, latent_w=40), [1 << 16, 1 << 16], 20, 4),
    ("c5red_5gpu_odd", "pixart_alpha", dict(depth=2, latent_h=32, latent_w=40),
     [1 << 16, 3 << 14, 1 << 15, 1 << 16, 1 << 12], 20, 4),
]
_cache = {}


def _inputs(name, **kw):
    key = (name, tuple(sorted((k, str(v)) for k, v in kw.items())))
    if key not in _cache:
        cfg = configs.model(name, **kw)
        _cache[key] = (cfg, gen.weights(cfg), gen.noise(cfg), gen.cond(cfg))
    return _cache[key]


def _split(cfg, speed, mb, mw):
    u = configs.rows_per_unit(cfg)
    return OP.plan_cfg_split(speed, mb, mw, cfg["latent_h"] // u, u)


def _oracle(cfg, W, x, c, plan, dtype):
    key = dict(kind="stadi_run", cfg=cfg, dtype=dtype, plan=plan)
    return refcache.cached(key, lambda: OR.run(cfg, gen.weights_bf16(W) if dtype == 0 else W,
                                               x, c, plan))


def oracle_cases():
    for _, name, kw, speed, mb, mw in CASES:
        cfg, W, x, c = _inputs(name, **kw)
        yield cfg, W, x, c, _split(cfg, speed, mb, mw)["pair_plan"], 0


@pytest.fixture(scope="module")
def S():
    from paper_2509_04719_b200 import stadi
    return stadi


def _desc(S, name, cfg):
    return S.model_desc(name, 0, depth=cfg["depth"], latent_h=cfg["latent_h"],
                        latent_w=cfg["latent_w"])


def _local(S, name, cfg, W, x, c, speed, mb, mw):
    ctx = S.Context(_desc(S, name, cfg), n_local=len(speed))
    try:
        ctx.load_weights([W[k] for k, _, _ in configs.manifest(cfg)])
        u = configs.rows_per_unit(cfg)
        p = S.plan(speed, mb, mw, cfg["latent_h"] // u, u, flags=S.CFG_SPLIT)
        outs = []
        for _ in range(2):
            out = np.zeros_like(x)
            ctx.run(p, x, c, out)
            outs.append(out)
        assert np.array_equal(outs[0], outs[1])
        return outs[0], p
    finally:
        ctx.close()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_cfg_split_local(S, case):
    cid, name, kw, speed, mb, mw = case
    cfg, W, x, c = _inputs(name, **kw)
    sp = _split(cfg, speed, mb, mw)
    got, p = _local(S, name, cfg, W, x, c, speed, mb, mw)
    d = p.to_dict()
    for k in ("tier", "steps", "rows", "branch", "partner"):
        assert d[k] == sp[k], k
    ref = _oracle(cfg, W, x, c, sp["pair_plan"], 0)
    err = float(np.max(np.abs(got.astype(np.float64) - ref)) / np.max(np.abs(ref)))
    print(f"CFG-split {cid}: pairs {sp['pairs']} steps={d['steps']} rows={d['rows']} "
          f"max-abs-rel={err:.3e}")
    assert err <= TOL


def test_cfg_split_ipc_and_vgpu(S):
    """The C2 4-GPU split as 4 processes on one GPU (IPC): the same bits as local mode;
    as 4 virtual GPUs of 24 SMs: within tolerance of the oracle (a 24-SM persistent
    grid picks other split-K factors, so the fp32 summation order differs)."""
    from paper_2509_04719_b200.vgpu import VirtualGpus
    _, name, kw, speed, mb, mw = CASES[0]
    cfg, W, x, c = _inputs(name, **kw)
    loc, p = _local(S, name, cfg, W, x, c, speed, mb, mw)
    world = len(speed)
    sess = S.ipc_session_id()[:16].hex()
    with tempfile.TemporaryDirectory() as d:
        procs = [subprocess.Popen([sys.executable, WORKER, d, str(r), str(world), sess, name, "0",
                                   ",".join(map(str, speed)), str(mb), str(mw), str(S.CFG_SPLIT),
                                   json.dumps(kw), "2"],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
                 for r in range(world)]
        try:
            logs = [pr.communicate(timeout=420)[0] for pr in procs]
        finally:
            for pr in procs:
                if pr.poll() is None:
                    pr.kill()
        for r, pr in enumerate(procs):
            assert pr.returncode == 0, logs[r][-3000:]
        outs = [np.load(os.path.join(d, f"rank{r}.npy")) for r in range(world)]
    for r in range(world):
        assert np.array_equal(outs[r][-1], loc), r
    vg = VirtualGpus(_desc(S, name, cfg), world, 24, [W[k] for k, _, _ in configs.manifest(cfg)])
    try:
        vo = [np.zeros_like(x) for _ in range(world)]
        vg.call("run", p, x, c, per_rank=lambda r: {"out": vo[r]})
    finally:
        vg.close()
    ref = _oracle(cfg, W, x, c, _split(cfg, speed, mb, mw)["pair_plan"], 0)
    for r in range(world):
        assert np.array_equal(vo[r], vo[0]), r
    err = float(np.max(np.abs(vo[0].astype(np.float64) - ref)) / np.max(np.abs(ref)))
    print(f"CFG-split C2 4 ranks: IPC processes == local mode; virtual GPUs max-abs-rel={err:.3e}")
    assert err <= TOL
