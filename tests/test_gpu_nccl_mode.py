"""NCCL-mode code path on one GPU (GPU tests).

gpurun provides one GPU and NCCL refuses two ranks on one device, so the
multi-process exchange cannot run here.  STADI_FORCE_NCCL=1 makes a world == 1,
n_local == 1 context run the NCCL-mode code path with a single-rank communicator:
the exchange publishes by (grouped) ncclBroadcast on the high-priority comm
stream, readers wait on the per-(site, version parity) events, the final gather
is an NCCL broadcast per band, profiling all-gathers its time, and no CUDA graphs
are used.  Its output must equal local mode bit for bit (same kernels, same
order of arithmetic) and the oracle within the north-star tolerance.
"""
import os

import numpy as np
import pytest

from oracle import stadi as OR
from synth import configs, gen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {0: 2e-2, 1: 1e-4}


@pytest.fixture(scope="module")
def S():
    from paper_2509_04719_b200 import stadi
    return stadi


def _run(S, name, cfg, W, x, c, mb, mw, dtype, nccl):
    old = os.environ.get("STADI_FORCE_NCCL")
    os.environ["STADI_FORCE_NCCL"] = "1" if nccl else "0"
    try:
        desc = S.model_desc(name, dtype, depth=cfg.get("depth", 0) if name != "tiny_unet" else 0,
                            latent_h=cfg["latent_h"], latent_w=cfg["latent_w"])
        ctx = S.Context(desc, n_local=1)
    finally:
        if old is None:
            del os.environ["STADI_FORCE_NCCL"]
        else:
            os.environ["STADI_FORCE_NCCL"] = old
    try:
        ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
        ms, sp = ctx.profile_warmup(2, 1)
        assert ms[0] > 0 and sp[0] == 1 << 20
        u = configs.rows_per_unit(cfg)
        p = S.plan([1 << 20], mb, mw, cfg["latent_h"] // u, u)
        outs = []
        for dev in (False, True):
            if dev:
                noise = torch.from_numpy(x).cuda()
                out = torch.zeros_like(noise)
                ctx.run(p, noise, c, out)
                outs.append(out.cpu().numpy().astype(np.float64))
            else:
                out = np.zeros_like(x)
                ctx.run(p, x, c, out)
                outs.append(out.astype(np.float64))
        assert np.array_equal(outs[0], outs[1])
        return outs[0]
    finally:
        ctx.close()


CASES = [("tiny_dit", {}, 10, 2, 1), ("tiny_dit", {}, 10, 2, 0), ("tiny_unet", {}, 6, 2, 0),
         ("dit_xl2", dict(depth=2), 10, 4, 0)]


@pytest.mark.parametrize("name,kw,mb,mw,dtype", CASES)
def test_nccl_mode_single_rank(S, name, kw, mb, mw, dtype):
    cfg = configs.model(name, **kw)
    W, x, c = gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)
    got = _run(S, name, cfg, W, x, c, mb, mw, dtype, nccl=True)
    loc = _run(S, name, cfg, W, x, c, mb, mw, dtype, nccl=False)
    assert np.array_equal(got, loc), "NCCL mode must equal local mode bit for bit"
    ref = OR.sequential(cfg, gen.weights_bf16(W) if dtype == 0 else W, x, c, mb)
    err = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
    print(f"NCCL-mode {name} dtype={dtype} max-abs-rel={err:.3e}")
    assert err <= TOL[dtype]


def test_nccl_mode_emulator(S):
    """The bench's N > 1 order on the NCCL path: probe, emulator, probe, run, stop."""
    cfg = configs.model("tiny_dit")
    W, x, c = gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)
    os.environ["STADI_FORCE_NCCL"] = "1"
    try:
        ctx = S.Context(S.model_desc("tiny_dit", 0), n_local=1)
    finally:
        del os.environ["STADI_FORCE_NCCL"]
    try:
        ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
        ctx.profile_warmup(1, 1)
        # created before the emulator: torch's first stream-pool use synchronises
        # the device, which would wait for the emulator's resident kernel
        st = torch.cuda.Stream()
        ctx.emulator_start(50)
        ctx.profile_warmup(2, 1)
        out = np.zeros_like(x)
        ctx.run(S.plan([1 << 20], 10, 2, 8, 2), x, c, out, stream=st)
        ctx.emulator_stop()
        assert np.all(np.isfinite(out))
    finally:
        ctx.close()
