"""Pins for the DDPM (eta = 1) sampler variant (R19, oracle/diffusion.py
ddpm_step) and its counter-based noise generator (synth/gen.py ddpm_noise).

* Consecutive timesteps: the step is the DDPM ancestral step of ref. [1]
  (Ho et al. Eq. 7): mean = mu_tilde(x_t, x0_hat) =
  sqrt(abar_{t-1}) beta_t / (1 - abar_t) x0 + sqrt(1 - beta_t)(1 - abar_{t-1})
  / (1 - abar_t) x_t, std = sqrt(beta_tilde_t), beta_tilde_t =
  (1 - abar_{t-1}) / (1 - abar_t) beta_t.  Written out here from [1], not
  from the oracle's [28] Eq. 12 form.
* Marginal preservation (exact): with eps the true noise of x_t = alpha x0 +
  sigma n, the eps- and z-coefficients' squares sum to 1 - abar'.
* Exact data point: x_t on the data manifold with the true eps and z = 0 moves
  along the posterior mean.
* Patch-parallel with fresh exchange equals the unpatched DDPM run (the z of a
  band is the band's rows of the full-image z_m).
* The generator: Philox4x64-10 known-answer block (Random123 KAT, key 0,
  counter 0), N(0, 1) moments and a KS test.
"""
import numpy as np
import pytest
from scipy import stats

from oracle import diffusion, schedule, stadi
from synth import configs, gen


@pytest.mark.parametrize("kind", ["linear", "scaled_linear"])
def test_ddpm_consecutive_is_ho_posterior(kind):
    ab = diffusion.alpha_bar(kind)
    rng = np.random.default_rng(7)
    x, e, z = rng.standard_normal((3, 64))
    for t in (999, 500, 37, 1):
        beta = 1.0 - ab[t] / ab[t - 1]
        x0 = (x - np.sqrt(1 - ab[t]) * e) / np.sqrt(ab[t])
        mean = (np.sqrt(ab[t - 1]) * beta / (1 - ab[t]) * x0
                + np.sqrt(1 - beta) * (1 - ab[t - 1]) / (1 - ab[t]) * x)
        std = np.sqrt((1 - ab[t - 1]) / (1 - ab[t]) * beta)
        got = diffusion.ddpm_step(ab, x, e, t, t - 1, z)
        np.testing.assert_allclose(got, mean + std * z, rtol=0, atol=1e-12)


def test_ddpm_preserves_marginal_variance():
    """x' = c_x x0 + c_e n + c_z z must have c_x = alpha' and c_e^2 + c_z^2 = 1 - abar'."""
    ab = diffusion.alpha_bar("scaled_linear")
    g = schedule.fast_grid(50)
    for m in (0, 10, 48):
        t = g[m]
        for tp in (g[m + 1], g[m + 2] if m + 2 < 50 else schedule.FINAL):
            ab2 = ab[0] if tp < 0 else ab[tp]
            a, s = np.sqrt(ab[t]), np.sqrt(1 - ab[t])
            one = np.ones(1)
            zero = np.zeros(1)
            cx = diffusion.ddpm_step(ab, a * one, zero, t, tp, zero)[0]      # x0 = 1, n = 0
            ce = diffusion.ddpm_step(ab, s * one, one, t, tp, zero)[0]       # x0 = 0, n = 1
            cz = diffusion.ddpm_step(ab, zero, zero, t, tp, one)[0]
            assert abs(cx - np.sqrt(ab2)) < 1e-12
            assert abs(ce ** 2 + cz ** 2 - (1 - ab2)) < 1e-12
            assert cz > 0


def test_ddpm_without_noise_term_is_not_ddim():
    """eta = 1 differs from Eq. 3 (a dropped sigma_eta^2 inside the eps
    coefficient would make them coincide at z = 0)."""
    ab = diffusion.alpha_bar("linear")
    x, e = np.ones(4), np.full(4, 0.5)
    a = diffusion.ddpm_step(ab, x, e, 500, 480, np.zeros(4))
    b = diffusion.ddim_step(ab, x, e, 500, 480)
    assert np.max(np.abs(a - b)) > 1e-4


def test_philox_kat_and_normal_moments():
    w = gen.philox_words(0, 0, 4)
    assert [int(v) for v in w] == [0x16554d9eca36314c, 0xdb20fe9d672d0fdc,
                                   0xd7e772cee186176b, 0x7e68b68aec7ba23b]
    z = gen.ddpm_noise((128, 128, 4), 5)
    assert abs(z.mean()) < 0.01 and abs(z.var() - 1) < 0.01
    assert stats.kstest(z.ravel(), "norm").pvalue > 1e-3
    # distinct m give independent draws; same m reproduces
    assert np.array_equal(z, gen.ddpm_noise((128, 128, 4), 5))
    assert abs(np.corrcoef(z.ravel(), gen.ddpm_noise((128, 128, 4), 6).ravel())[0, 1]) < 0.01


def _c1():
    cfg = configs.model("tiny_dit")
    return cfg, gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)


def _zf(cfg):
    shape = (cfg["latent_h"], cfg["latent_w"], cfg["c_in"])
    return lambda m: gen.ddpm_noise(shape, m)


def test_ddpm_fresh_patch_run_equals_unpatched():
    cfg, W, x, c = _c1()
    seq = stadi.sequential(cfg, W, x, c, 10, ddpm_z=_zf(cfg))
    assert np.max(np.abs(seq - stadi.sequential(cfg, W, x, c, 10))) > 1e-3
    for speed in ([1, 1], [3, 2, 1]):
        p = stadi.plan_for(cfg, speed, 10, 10, flags=1)
        out = stadi.run(cfg, W, x, c, p, ddpm_z=_zf(cfg))
        assert np.max(np.abs(out - seq)) / np.max(np.abs(seq)) < 1e-12


def test_ddpm_single_gpu_run_is_sequential():
    cfg, W, x, c = _c1()
    out = stadi.run(cfg, W, x, c, stadi.plan_for(cfg, [1], 10, 2), ddpm_z=_zf(cfg))
    assert np.array_equal(out, stadi.sequential(cfg, W, x, c, 10, ddpm_z=_zf(cfg)))
