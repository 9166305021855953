"""Pins of the R34 multistep DPM-Solver-2 (oracle/diffusion.py dpm2m_step) -- CPU.

* Convergence order on the Gaussian toy whose diffusion ODE is solvable in closed
  form: data x0 ~ N(0, s^2) gives the exact noise prediction
  eps(x, t) = sigma_t x / (alpha_t^2 s^2 + sigma_t^2) and the exact flow map
  x(t') = sqrt((alpha'^2 s^2 + sigma'^2) / (alpha^2 s^2 + sigma^2)) x(t).  Eq. 3
  (DPM-Solver-1 = DDIM) must converge with order 1 (error halves when M doubles),
  the multistep solver with order 2 (error / 4) -- a dropped history term, a wrong
  r or sign falls back to order 1 or diverges.
* With a constant eps the history term vanishes: the step equals Eq. 3 exactly;
  the first step of a band (no history) is Eq. 3.
* Protocol: N = 1 equals the sequential solver; with time-invariant activations
  (constant eps) any stale plan equals the sequential run.
"""
import math

import numpy as np

from oracle import diffusion, schedule
from oracle import stadi as OR
from synth import configs, gen


def _toy_error(m_base, solver, s=0.7):
    ab = diffusion.alpha_bar("linear")
    grid = schedule.fast_grid(m_base) + [schedule.FINAL]

    def a_s(t):
        a, sg, _ = diffusion.alpha_sigma(ab, t)
        return a, sg
    x = 1.3
    hist = None
    for m in range(m_base):
        t, tp = grid[m], grid[m + 1]
        a, sg = a_s(t)
        eps = sg * x / (a * a * s * s + sg * sg)
        if solver == "ddim":
            x = diffusion.ddim_step(ab, x, eps, t, tp)
        else:
            x, hist = diffusion.dpm2m_step(ab, x, eps, t, tp, hist), (eps, t)
    a0, s0 = a_s(grid[0])
    a1, s1 = a_s(schedule.FINAL)
    exact = 1.3 * math.sqrt((a1 * a1 * s * s + s1 * s1) / (a0 * a0 * s * s + s0 * s0))
    return abs(x - exact)


def test_convergence_orders_gaussian_toy():
    e1 = [_toy_error(m, "ddim") for m in (25, 50, 100)]
    e2 = [_toy_error(m, "dpm2m") for m in (25, 50, 100)]
    for a, b in zip(e1, e1[1:]):
        assert 1.7 < a / b < 2.4, e1                 # first order
    for a, b in zip(e2, e2[1:]):
        assert 3.2 < a / b < 5.0, e2                 # second order
    assert e2[-1] < e1[-1] / 5


def test_constant_eps_and_first_step_reduce_to_eq3():
    ab = diffusion.alpha_bar("scaled_linear")
    rng = np.random.default_rng(0)
    x, eps = rng.standard_normal((2, 5, 3))
    for t, tp, s_prev in ((901, 801, 961), (101, 1, 201), (21, schedule.FINAL, 41)):
        ref = diffusion.ddim_step(ab, x, eps, t, tp)
        assert np.array_equal(diffusion.dpm2m_step(ab, x, eps, t, tp, None), ref)
        got = diffusion.dpm2m_step(ab, x, eps, t, tp, (eps.copy(), s_prev))
        assert np.allclose(got, ref, rtol=0, atol=1e-12)
        # and a changing eps does change it
        got2 = diffusion.dpm2m_step(ab, x, eps, t, tp, (eps + 0.1, s_prev))
        assert np.max(np.abs(got2 - ref)) > 1e-4


def test_dpm2m_protocol_reductions():
    cfg = configs.model("tiny_dit")
    W, x, c = gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)
    seq = OR.sequential(cfg, W, x, c, 10, sampler="dpm2m")
    assert np.array_equal(OR.run(cfg, W, x, c, OR.plan_for(cfg, [1], 10, 2), sampler="dpm2m"), seq)
    assert np.max(np.abs(seq - OR.sequential(cfg, W, x, c, 10))) > 1e-6   # not DDIM
    W = dict(W)
    for k in ("x_embed.w", "t_embed.w1", "t_embed.w2"):
        W[k] = np.zeros_like(W[k])
    seq = OR.sequential(cfg, W, x, c, 10, sampler="dpm2m")
    for speed in ([2, 1], [3, 2, 1]):
        p = OR.plan_for(cfg, speed, 10, 2)
        out = OR.run(cfg, W, x, c, p, sampler="dpm2m")
        assert np.max(np.abs(out - seq)) <= 1e-12 * np.max(np.abs(seq)), speed
