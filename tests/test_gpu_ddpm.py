"""DDPM (eta = 1) sampler parity on the GPU (R19; north star "fused DDIM/DDPM
sampler update").

* stadi_k_ddpm_noise: the in-kernel counter-based generator against
  synth/gen.py's numpy Philox4x64-10 + Box-Muller, element by element over a
  ragged range starting mid-block (the only difference is fp32 vs fp64
  rounding of the Box-Muller transform).
* stadi_k_sampler: the fused CFG + unpatchify + DDPM update of a band against
  oracle/diffusion.py ddpm_step on the oracle's unpatchify of eps.
* End to end (stadi_run, local mode) against oracle.stadi.run with the same
  z_m: C1 tiny DiT (fp32 debug and bf16; tier-2 rank = stride-2 jumps), the C2
  DiT-XL/2 shape depth-reduced, and the tiny U-Net.
"""
import numpy as np
import pytest

from oracle import diffusion, schedule
from oracle import stadi as OR
from synth import configs, gen
import refcache

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {0: 2e-2, 1: 1e-4}
SEED = gen.SEED_DDPM


@pytest.fixture(scope="module")
def S():
    from paper_2509_04719_b200 import stadi
    return stadi


def test_ddpm_noise_generator(S):
    shape = (64, 48, 4)
    n0 = int(np.prod(shape))
    e0 = 4 * 333 + 3                                  # start mid counter block
    n = n0 - e0 - 5                                   # ragged end
    for m in (0, 7, 49):
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        S.k_ddpm_noise(out, n, SEED, m, e0)
        ref = gen.ddpm_noise(shape, m, SEED).ravel()[e0:e0 + n]
        got = out.cpu().numpy().astype(np.float64)
        assert np.max(np.abs(got - ref)) < 2e-5, m


@pytest.mark.parametrize("p,B", [(2, 2), (1, 2), (2, 1)])
def test_sampler_kernel_ddpm(S, p, B):
    rng = np.random.default_rng(3)
    H, W, C, c_out, row0 = 12, 20, 4, 8, 6           # band rows [6, 18) of a 32-row image
    ld = p * p * c_out + 8
    ntok = (H // p) * (W // p)
    x = rng.standard_normal((H, W, C)).astype(np.float32)
    eps_raw = rng.standard_normal((ntok * B, ld)).astype(np.float32)
    g = 4.5
    ab = diffusion.alpha_bar("linear")
    grid = schedule.fast_grid(20)
    m, t, tp = 5, grid[5], grid[7]
    # oracle: unpatchify + CFG + ddpm_step on the band's rows of z_m
    e = np.zeros((H, W, C))
    for r in range(H):
        for c_ in range(W):
            tok = (r // p) * (W // p) + c_ // p
            j = ((r % p) * p + c_ % p) * c_out
            eu = eps_raw[tok * B + 0, j:j + C].astype(np.float64)
            e[r, c_] = eu if B == 1 else eu + g * (eps_raw[tok * B + 1, j:j + C] - eu)
    z = gen.ddpm_noise((32, W, C), m, SEED)[row0:row0 + H]
    ref = diffusion.ddpm_step(ab, x.astype(np.float64), e, t, tp, z)
    # coefficients as the runtime computes them (fp64 -> fp32)
    a1, a2 = ab[t], ab[tp]
    se = np.sqrt((1 - a2) / (1 - a1)) * np.sqrt(1 - a1 / a2)
    A = np.sqrt(a2) / np.sqrt(a1)
    Bc = np.sqrt(1 - a2 - se * se) - np.sqrt(a2) * np.sqrt(1 - a1) / np.sqrt(a1)
    xd = torch.from_numpy(x).cuda()
    ed = torch.from_numpy(eps_raw).cuda()
    S.k_sampler(xd, ed, H, W, C, p, c_out, ld, B, g, A, Bc, se, SEED, m, row0)
    got = xd.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-5


_cache = {}


def _inputs(name, **kw):
    key = (name, tuple(sorted((k, str(v)) for k, v in kw.items())))
    if key not in _cache:
        cfg = configs.model(name, **kw)
        _cache[key] = (cfg, gen.weights(cfg), gen.noise(cfg), gen.cond(cfg))
    return _cache[key]


def _zf(cfg, seed=SEED):
    shape = (cfg["latent_h"], cfg["latent_w"], cfg["c_in"])
    return lambda m: gen.ddpm_noise(shape, m, seed)


def _oracle(cfg, W, x, c, plan, dtype, seed=SEED):
    key = dict(kind="stadi_run_ddpm", seed=seed, cfg=cfg, dtype=dtype, plan=plan)

    def compute():
        return OR.run(cfg, gen.weights_bf16(W) if dtype == 0 else W, x, c, plan,
                      ddpm_z=_zf(cfg, seed))
    return refcache.cached(key, compute)


CASES = [("tiny_dit", {}, [1 << 20, 1 << 19], 10, 2),
         ("dit_xl2", dict(depth=2), [65536, 39322], 50, 4),
         ("tiny_unet", {}, [1 << 20, 1 << 19], 10, 2)]


def oracle_cases():
    for name, kw, speed, mb, mw in CASES:
        for dtype in ((1, 0) if name == "tiny_dit" else (0,)):
            cfg, W, x, c = _inputs(name, **kw)
            yield cfg, W, x, c, OR.plan_for(cfg, speed, mb, mw), dtype
    for name in ("tiny_dit", "tiny_unet"):          # the second request's seed
        cfg, W, x, c = _inputs(name)
        yield cfg, W, x, c, OR.plan_for(cfg, [1 << 20, 1 << 19], 10, 2), 0, SEED + 1


def _gpu_run(S, name, cfg, W, x, c, speed, mb, mw, dtype):
    desc = S.model_desc(name, dtype, depth=cfg.get("depth", 0) if name != "tiny_unet" else 0,
                        latent_h=cfg["latent_h"], latent_w=cfg["latent_w"],
                        sampler=S.SAMPLER_DDPM)
    ctx = S.Context(desc, n_local=len(speed))
    try:
        ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
        u = configs.rows_per_unit(cfg)
        p = S.plan(speed, mb, mw, cfg["latent_h"] // u, u)
        out = np.zeros_like(x)
        ctx.run(p, x, dict(c, ddpm_seed=SEED), out)
        return out.astype(np.float64), p
    finally:
        ctx.close()


@pytest.mark.parametrize("name,kw,speed,mb,mw,dtype",
                         [(n, k, s, a, b, d) for n, k, s, a, b in CASES
                          for d in ((1, 0) if n == "tiny_dit" else (0,))])
def test_ddpm_run(S, name, kw, speed, mb, mw, dtype):
    cfg, W, x, c = _inputs(name, **kw)
    plan = OR.plan_for(cfg, speed, mb, mw)
    ref = _oracle(cfg, W, x, c, plan, dtype)
    got, p = _gpu_run(S, name, cfg, W, x, c, speed, mb, mw, dtype)
    assert p.to_dict()["steps"] == plan["steps"]
    assert np.all(np.isfinite(got))
    err = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    print(f"DDPM {name} dtype={dtype} max-abs-rel={err:.3e}")
    assert err <= TOL[dtype]


@pytest.mark.parametrize("name", ["tiny_dit", "tiny_unet"])
def test_ddpm_seed_changes_between_requests(S, name):
    """Two requests on ONE context and plan with different DDPM seeds: the step
    graphs captured by the first request must draw the second request's z_m
    (the sampler reads the key from device memory), each against the oracle."""
    cfg, W, x, c = _inputs(name)
    speed, mb, mw = [1 << 20, 1 << 19], 10, 2
    plan = OR.plan_for(cfg, speed, mb, mw)
    desc = S.model_desc(name, 0, latent_h=cfg["latent_h"], latent_w=cfg["latent_w"],
                        sampler=S.SAMPLER_DDPM)
    ctx = S.Context(desc, n_local=2)
    try:
        ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
        u = configs.rows_per_unit(cfg)
        p = S.plan(speed, mb, mw, cfg["latent_h"] // u, u)
        outs = []
        for seed in (SEED, SEED + 1, SEED):
            out = np.zeros_like(x)
            ctx.run(p, x, dict(c, ddpm_seed=seed), out)
            outs.append(out.astype(np.float64))
    finally:
        ctx.close()
    assert np.array_equal(outs[0], outs[2])
    for seed, got in ((SEED, outs[0]), (SEED + 1, outs[1])):
        ref = _oracle(cfg, W, x, c, plan, 0, seed)
        err = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
        print(f"DDPM two-request {name} seed={seed} max-abs-rel={err:.3e}")
        assert err <= TOL[0]
