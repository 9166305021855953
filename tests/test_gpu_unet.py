"""U-Net family end-to-end parity (GPU): STADI through the C ABI (local mode,
all ranks of the plan on one GPU) against the fp64 oracle (oracle/unet.py via
oracle.stadi.run) on identical seeded inputs.  Exercises every U-Net exchange
site kind: self-attention K/V, 3x3-conv halos (stride 1, stride 2 and the
pre-upsample rows), GroupNorm partial statistics (R15-R17).

Tolerances (north star): max-abs-rel <= 1e-4 fp32 debug build, <= 2e-2 bf16.
Reduced variants keep the widths / heads / level structure of C3 (SD-1.5) and
C4 (SDXL) but use a 32x32 latent and transformer depth <= 1 so the oracle
finishes in seconds.
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
_cache = {}

SD15_KW = dict(latent_h=32, latent_w=32)
SDXL_KW = dict(latent_h=32, latent_w=32, tdepth=[0, 1, 1], mid_depth=1)
TINY_CASES = [([1 << 20, 1 << 19], 0, 10, 2),          # tier 1 / tier 2 (C1-like)
              ([3, 2, 1], OP.NO_TA | OP.NO_SA, 6, 2),   # uniform patch parallelism
              ([1], 0, 4, 2),                            # single GPU == sequential
              ([5, 4, 1], 0, 6, 2)]                      # an excluded GPU


def _inputs(name, **kw):
    key = (name, tuple(sorted((k, str(v)) for k, v in kw.items())))
    if key not in _cache:
        cfg = configs.model(name, **kw)
        _cache[key] = (cfg, gen.weights(cfg), gen.noise(cfg), gen.cond(cfg))
    return _cache[key]


def _oracle(cfg, W, x, c, plan, dtype):
    key = dict(kind="stadi_run", cfg=cfg, dtype=dtype, plan=plan)

    def compute():
        return OR.run(cfg, gen.weights_bf16(W) if dtype == 0 else W, x, c, plan)
    return refcache.cached(key, compute)


def oracle_cases():
    for dtype in (1, 0):
        cfg, W, x, c = _inputs("tiny_unet")
        for speed, flags, mb, mw in TINY_CASES:
            yield cfg, W, x, c, OR.plan_for(cfg, speed, mb, mw, flags=flags), dtype
    for name, kw in (("sd15", SD15_KW), ("sdxl", SDXL_KW)):
        cfg, W, x, c = _inputs(name, **kw)
        yield cfg, W, x, c, OR.plan_for(cfg, [65536, 39322], 6, 2), 0


@pytest.fixture(scope="module")
def S():
    from paper_2509_04719_b200 import stadi
    return stadi


def _gpu_run(S, name, cfg, W, x, c, speed, mb, mw, dtype, flags=0, depth=0):
    desc = S.model_desc(name, dtype, depth=depth, latent_h=cfg["latent_h"],
                        latent_w=cfg["latent_w"])
    ctx = S.Context(desc, n_local=len(speed))
    try:
        ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
        u = configs.rows_per_unit(cfg)
        p = S.plan(speed, mb, mw, cfg["latent_h"] // u, u, flags=flags)
        out = np.zeros_like(x)
        st = ctx.run(p, x, c, out)
        return out.astype(np.float64), p, st
    finally:
        ctx.close()


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.mark.parametrize("dtype", [1, 0], ids=["fp32", "bf16"])
@pytest.mark.parametrize("speed,flags,mb,mw", TINY_CASES)
def test_tiny_unet(S, dtype, speed, flags, mb, mw):
    cfg, W, x, c = _inputs("tiny_unet")
    plan = OR.plan_for(cfg, speed, mb, mw, flags=flags)
    ref = _oracle(cfg, W, x, c, plan, dtype)
    got, p, st = _gpu_run(S, "tiny_unet", cfg, W, x, c, speed, mb, mw, dtype, flags=flags)
    assert p.to_dict()["rows"] == plan["rows"] and p.to_dict()["steps"] == plan["steps"]
    assert np.all(np.isfinite(got))
    err = _rel(got, ref)
    print(f"tiny_unet {speed} dtype={dtype} max-abs-rel={err:.3e} launches={st.kernel_launches}")
    assert err <= TOL[dtype]


@pytest.mark.parametrize("name,kw,depth", [("sd15", SD15_KW, 0), ("sdxl", SDXL_KW, 1)])
def test_c3_c4_reduced_bf16(S, name, kw, depth):
    """C3 / C4 shapes (widths, heads, levels, CFG, scaled-linear schedule) on a
    32x32 latent, transformer depth <= 1; 2 GPUs, the second at 40% occupancy
    (v = 0.6 -> steps [6, 4])."""
    cfg, W, x, c = _inputs(name, **kw)
    plan = OR.plan_for(cfg, [65536, 39322], 6, 2)
    ref = _oracle(cfg, W, x, c, plan, 0)
    got, p, _ = _gpu_run(S, name, cfg, W, x, c, [65536, 39322], 6, 2, 0, depth=depth)
    assert np.all(np.isfinite(got))
    err = _rel(got, ref)
    print(f"{name}(reduced) bf16 max-abs-rel={err:.3e}")
    assert err <= TOL[0]
