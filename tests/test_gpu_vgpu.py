"""Virtual GPUs (GPU): the ranks of a request run CONCURRENTLY on one B200, each in
its own green-context SM partition (stadi_dist_desc.vgpu_sms), one host thread per
rank, exchanging over the IPC transport (in-process peers: the QKV epilogue stores
into the other partition's slots, flags by stream memory operations).

Checks, as for the multi-process test: every rank gathers the same latent, equal
bit for bit to the local-mode run (all ranks lock-step in one context), and within
the north-star tolerance of the fp64 oracle; the occupancy emulator may hold part of
a partition without changing the result.
"""
import numpy as np
import pytest

from oracle import planner as OP
from oracle import stadi as OR
from synth import configs, gen
import refcache

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {0: 2e-2, 1: 1e-4}
CASES = [  # id, name, kwargs, speeds, m_base, m_warmup, flags, sms, occupancy
    ("c1_tier2", "tiny_dit", {}, [1 << 20, 1 << 19], 10, 2, 0, 32, None),
    ("c1_excluded_4", "tiny_dit", {}, [100, 60, 100, 10], 10, 2, 0, 24, None),
    ("unet_3", "tiny_unet", {}, [3, 2, 1], 6, 2, OP.NO_TA | OP.NO_SA, 32, None),
    ("c2_depth2", "dit_xl2", dict(depth=2), [65536, 39322], 50, 4, 0, 56, None),
    ("c2_depth2_emu40", "dit_xl2", dict(depth=2), [65536, 39322], 50, 4, 0, 56, [0, 40]),
]


@pytest.fixture(scope="module")
def S():
    from paper_2509_04719_b200 import stadi
    return stadi


def _oracle(cfg, W, x, c, plan, dtype):
    key = dict(kind="stadi_run", cfg=cfg, dtype=dtype, plan=plan)
    return refcache.cached(key, lambda: OR.run(cfg, gen.weights_bf16(W) if dtype == 0 else W,
                                               x, c, plan))


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_virtual_gpus(S, case):
    from paper_2509_04719_b200.vgpu import VirtualGpus
    cid, name, kw, speed, mb, mw, flags, sms, occ = case
    n = len(speed)
    cfg = configs.model(name, **kw)
    W, x, c = gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)
    depth = cfg.get("depth", 0) if cfg["family"] == "dit" else 0
    desc = S.model_desc(name, 0, depth=depth, latent_h=cfg["latent_h"], latent_w=cfg["latent_w"])
    u = configs.rows_per_unit(cfg)
    p = S.plan(speed, mb, mw, cfg["latent_h"] // u, u, flags=flags)
    vg = VirtualGpus(desc, n, sms, [W[k] for k, _, _ in configs.manifest(cfg)])
    try:
        vg.call("profile_warmup", 2, n)
        if occ:
            vg.call("emulator_start", per_rank=lambda r: {"pct": occ[r]})
        outs = [np.zeros_like(x) for _ in range(n)]
        try:
            stats = None
            for _ in range(2):   # second request replays the captured step graphs
                stats = vg.call("run", p, x, c, per_rank=lambda r: {"out": outs[r]})
        finally:
            if occ:
                vg.call("emulator_stop")
    finally:
        vg.close()
    for r in range(n):
        assert np.array_equal(outs[r], outs[0]), r
    ctx = S.Context(desc, n_local=n)
    try:
        ctx.load_weights([W[k] for k, _, _ in configs.manifest(cfg)])
        loc = np.zeros_like(x)
        ctx.run(p, x, c, loc)
    finally:
        ctx.close()
    assert np.array_equal(outs[0], loc), "virtual GPUs must equal local mode bit for bit"
    plan = OR.plan_for(cfg, speed, mb, mw, flags=flags)
    ref = _oracle(cfg, W, x, c, plan, 0)
    err = float(np.max(np.abs(outs[0].astype(np.float64) - ref)) / np.max(np.abs(ref)))
    ms = [round(s.ms_total, 2) for s in stats]
    print(f"VGPU {cid}: {n} partitions x {sms} SMs occ={occ} steps={plan['steps']} "
          f"rows={plan['rows']} max-abs-rel={err:.3e} ms={ms} "
          f"graph_steps={[s.graph_steps for s in stats]}")
    assert err <= TOL[0]
