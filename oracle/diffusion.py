"""Oracle noise schedule and sampler update.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md L57 (Eq. 1): q(x_t|x_0) = N(alpha_t x_0, sigma_t^2 I).
PAPER.md L70-74 (Lemma 1, Eq. 3, DPM-Solver-1 == DDIM):
    x_{t_m} = (alpha_{t_m}/alpha_{t_{m-1}}) x_{t_{m-1}}
              - sigma_{t_m} (e^{h_m} - 1) eps_theta(x_{t_{m-1}}, t_{m-1}),
    h_m = lambda_{t_m} - lambda_{t_{m-1}},  lambda = log(alpha/sigma).
Readings:
  R18  alpha_bar_t = prod_{s<=t}(1 - beta_s), T = 1000; DiT shapes use the
       linear beta schedule [1e-4, 0.02], U-Net shapes scaled-linear
       [0.00085, 0.012]; alpha_t = sqrt(alpha_bar_t), sigma_t =
       sqrt(1 - alpha_bar_t); the "final" step lands on alpha_bar_0.
  R20  classifier-free guidance eps = eps_u + w (eps_c - eps_u).
"""
from __future__ import annotations

import numpy as np

T_TRAIN = 1000


def alpha_bar(kind: str, T: int = T_TRAIN) -> np.ndarray:
    """alpha_bar_t for t = 0..T-1 (R18)."""
    if kind == "linear":
        beta = np.linspace(1e-4, 0.02, T, dtype=np.float64)
    elif kind == "scaled_linear":
        beta = np.linspace(0.00085 ** 0.5, 0.012 ** 0.5, T, dtype=np.float64) ** 2
    else:
        raise ValueError(kind)
    return np.cumprod(1.0 - beta)


def alpha_sigma(abar: np.ndarray, t: int):
    """(alpha_t, sigma_t, lambda_t) of Eq. 1 / Lemma 1.  t = -1 means 'final'
    and uses alpha_bar_0 (R18)."""
    ab = abar[0] if t < 0 else abar[t]
    a = np.sqrt(ab)
    s = np.sqrt(1.0 - ab)
    return a, s, np.log(a / s)


def ddim_coeffs(abar: np.ndarray, t: int, t_prev: int):
    """Eq. 3 written as x' = A x + Bc eps:  A = alpha'/alpha,
    Bc = -sigma' (e^h - 1), h = lambda' - lambda."""
    a, s, lam = alpha_sigma(abar, t)
    a2, s2, lam2 = alpha_sigma(abar, t_prev)
    h = lam2 - lam
    return a2 / a, -s2 * np.expm1(h)


def ddim_step(abar, x, eps, t, t_prev):
    """Eq. 3 (L72)."""
    A, Bc = ddim_coeffs(abar, t, t_prev)
    return A * x + Bc * eps


def cfg_combine(eps_u, eps_c, w):
    """R20: eps = eps_u + w (eps_c - eps_u)."""
    return eps_u + w * (eps_c - eps_u)
