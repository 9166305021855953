"""GPU stale-exchange plumbing against an expectation that is not the oracle's
own stale run (GPU tests).

With every activation independent of x_t and t (DiT: patch- and t-embedding
weights zeroed; U-Net: conv_in and the time embedding zeroed), stale reads equal
fresh ones and eps is constant, so a STADI run with stale rounds and tier-2
stride-2 steps must reproduce the unpatched sequential run (pinned on the CPU in
tests/test_oracle_model.py / test_oracle_unet.py).  Here the CUDA path, local
mode (all ranks on one GPU, exchange by device copies), is compared with
oracle.stadi.sequential at the north-star tolerances.
"""
import numpy as np
import pytest

from oracle import stadi as OR
from synth import configs, gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {0: 2e-2, 1: 1e-4}
ZERO = {"tiny_dit": ("x_embed.w", "t_embed.w1", "t_embed.w2"),
        "tiny_unet": ("conv_in.w", "time.w1", "time.w2")}


@pytest.fixture(scope="module")
def S():
    from paper_2509_04719_b200 import stadi
    return stadi


@pytest.mark.parametrize("dtype", [1, 0], ids=["fp32", "bf16"])
@pytest.mark.parametrize("name,speed,mb,mw", [("tiny_dit", [2, 1], 10, 2),
                                              ("tiny_dit", [6, 1, 3], 10, 2),
                                              ("tiny_unet", [4, 2], 6, 2),
                                              ("tiny_unet", [6, 1, 3], 6, 2)])
def test_time_invariant_stale_run_equals_sequential(S, name, speed, mb, mw, dtype):
    cfg = configs.model(name)
    W, x, c = dict(gen.weights(cfg)), gen.noise(cfg), gen.cond(cfg)
    for k in ZERO[name]:
        W[k] = np.zeros_like(W[k])
    ctx = S.Context(S.model_desc(name, dtype), n_local=len(speed))
    try:
        ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
        u = configs.rows_per_unit(cfg)
        p = S.plan(speed, mb, mw, cfg["latent_h"] // u, u)
        assert any(t == 2 for t in p.to_dict()["tier"])          # a stride-2 rank
        out = np.zeros_like(x)
        ctx.run(p, x, c, out)
    finally:
        ctx.close()
    ref = OR.sequential(cfg, gen.weights_bf16(W) if dtype == 0 else W, x, c, mb)
    err = float(np.max(np.abs(out - ref)) / np.max(np.abs(ref)))
    print(f"{name} {speed} dtype={dtype} stale-vs-sequential max-abs-rel={err:.3e}")
    assert err <= TOL[dtype]
