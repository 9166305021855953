"""Pins of the U-Net oracle (oracle/unet.py) — CPU only.

What fixes the U-Net family independently of the oracle's own code:
* diffusers' published parameter counts of the SD-1.5 UNet (859,520,964) and the
  SDXL UNet (2,567,463,684) — an exact count pins every layer shape / channel
  bookkeeping of the architecture description (synth/configs.py);
* the up-path ResBlock input widths of SD-1.5 (its conv1 weight shapes);
* conv3x3 against a brute-force 7-deep loop; GroupNorm against a textbook
  formula; GELU(1) = Phi(1) = 0.8413447460685429; sinusoid closed forms;
* the patch protocol's reductions: with a fresh exchange (M_warmup = M_base)
  the band-parallel run equals the unpatched sequential run for any split
  (halos, GroupNorm partial sums, K/V, stride-2 and upsample halos all
  exercised), and N = 1 equals sequential DDIM.
"""
import math

import numpy as np
import pytest

from oracle import stadi as OR
from oracle import unet as OU
from synth import configs, gen


def _nparams(name):
    return sum(int(np.prod(s)) for _, s, _ in configs.manifest(configs.model(name)))


def test_sd15_param_count_matches_diffusers():
    assert _nparams("sd15") == 859_520_964


def test_sdxl_param_count_matches_diffusers():
    assert _nparams("sdxl") == 2_567_463_684


def test_sd15_up_path_resblock_inputs():
    io = OU.up_resnet_io(configs.model("sd15"))
    ins = [[a + b for a, b, _ in lv] for lv in io]
    assert ins == [[2560, 2560, 2560], [2560, 2560, 1920], [1920, 1280, 960], [960, 640, 640]]


def test_conv3x3_brute_force():
    rng = np.random.default_rng(0)
    for stride in (1, 2):
        xp = rng.standard_normal((2, 7, 9, 3))
        w = rng.standard_normal((4, 3, 3, 3))
        b = rng.standard_normal(4)
        got = OU.conv3x3_valid(xp, w, b, stride)
        Ho, Wo = (7 - 3) // stride + 1, (9 - 3) // stride + 1
        ref = np.zeros((2, Ho, Wo, 4))
        for n in range(2):
            for y in range(Ho):
                for x in range(Wo):
                    for o in range(4):
                        acc = b[o]
                        for c in range(3):
                            for ky in range(3):
                                for kx in range(3):
                                    acc += xp[n, stride * y + ky, stride * x + kx, c] * w[o, c, ky, kx]
                        ref[n, y, x, o] = acc
        assert np.allclose(got, ref, atol=1e-12)


def test_group_norm_partials_over_bands():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((2, 6, 5, 64)) * 3 + 1
    w, b = rng.standard_normal(64), rng.standard_normal(64)
    full = OU.group_norm_full(x, w, b, 1e-5)
    # textbook per-group formula by explicit loops on one group
    g = x[1, :, :, 4:6]
    mu, var = g.mean(), g.var()
    assert np.allclose(full[1, :, :, 4:6], (g - mu) / np.sqrt(var + 1e-5) * w[4:6] + b[4:6])
    # partial sums of three bands, summed, applied per band == full
    parts = [OU.gn_partials(x[:, a:bb]) for a, bb in ((0, 1), (1, 4), (4, 6))]
    tot = tuple(sum(p[i] for p in parts) for i in range(3))
    got = np.concatenate([OU.gn_apply(x[:, a:bb], tot, w, b, 1e-5)
                          for a, bb in ((0, 1), (1, 4), (4, 6))], axis=1)
    assert np.allclose(got, full, atol=1e-12)


def test_gelu_and_sinusoid_closed_forms():
    assert abs(OU.gelu_erf(np.array([1.0]))[0] - 0.8413447460685429) < 1e-15
    assert abs(OU.gelu_erf(np.array([-3.0]))[0] - (-3.0 * 0.5 * math.erfc(3 / math.sqrt(2)))) < 1e-15
    e = OU.timestep_sinusoid(0.0, 8)
    assert np.array_equal(e, [1, 1, 1, 1, 0, 0, 0, 0])
    e = OU.timestep_sinusoid(7.0, 4)          # f = [1, 10000^-1/2]
    assert np.allclose(e, [math.cos(7), math.cos(0.07), math.sin(7), math.sin(0.07)])


@pytest.fixture(scope="module")
def tiny():
    cfg = configs.model("tiny_unet")
    return cfg, gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)


@pytest.fixture(scope="module")
def tiny_seq(tiny):
    cfg, W, x, c = tiny
    return OR.sequential(cfg, W, x, c, 4)


@pytest.mark.parametrize("speed", [[1], [1, 1], [3, 2, 1], [5, 1, 4]])
def test_fresh_exchange_equals_unpatched(tiny, tiny_seq, speed):
    """M_warmup = M_base: every step exchanges fresh (R9) -> the band-parallel
    forward is exactly the unpatched forward, for every split (incl. an
    excluded rank and a 2-row band at the finest level)."""
    cfg, W, x, c = tiny
    p = OR.plan_for(cfg, speed, 4, 4)
    out = OR.run(cfg, W, x, c, p)
    assert np.max(np.abs(out - tiny_seq)) <= 1e-12 * np.max(np.abs(tiny_seq))


def test_stale_run_differs_but_stays_close(tiny, tiny_seq):
    """With stale exchange (M_warmup < M_base) the result is NOT sequential but
    close (Thm 1/2: O(1/M) deviation); a sanity bound, not a pin."""
    cfg, W, x, c = tiny
    p = OR.plan_for(cfg, [4, 2], 4, 2)
    assert p["steps"] == [4, 3]
    out = OR.run(cfg, W, x, c, p)
    d = np.max(np.abs(out - tiny_seq)) / np.max(np.abs(tiny_seq))
    assert 1e-9 < d < 0.5


def test_time_invariant_activations_make_staleness_exact(tiny):
    """Stale-protocol pin for the U-Net sites (K/V, conv halos incl. stride-2 and
    upsample rows, GroupNorm partial sums): with conv_in and the time embedding
    zeroed every activation is independent of x_t and t (the zero padding at the
    image borders still makes them vary over rows), so stale payloads equal fresh
    ones and eps is constant; any plan, stale rounds and stride-2 tier-2 steps
    included, must then reproduce the unpatched sequential run."""
    cfg, W, x, c = tiny
    W = dict(W)
    for k in ("conv_in.w", "time.w1", "time.w2"):
        W[k] = np.zeros_like(W[k])
    seq = OR.sequential(cfg, W, x, c, 6)
    assert np.std((seq - x)[:, :, 0], axis=0).max() > 0            # eps varies over rows
    for speed, flags in (([4, 2], 0), ([3, 2, 1], 1), ([5, 1, 4], 0), ([6, 1, 3], 0)):
        p = OR.plan_for(cfg, speed, 6, 2, flags=flags)
        out = OR.run(cfg, W, x, c, p)
        assert np.max(np.abs(out - seq)) <= 1e-12 * np.max(np.abs(seq)), (speed, flags)
