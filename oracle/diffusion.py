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
  R19  DDPM variant (north_star "fused DDIM/DDPM sampler update"; Eq. 2
       p_theta(x_{t-1}|x_t) = N(mu_theta, Sigma_theta) realised as the
       eta = 1 member of the DDIM family of ref. [28] (Song et al., Eq. 12),
       which for consecutive t equals the DDPM ancestral step of ref. [1]):
         x0_hat    = (x_t - sigma_t eps) / alpha_t
         sigma_eta = sqrt((1 - abar') / (1 - abar)) sqrt(1 - abar / abar')
         x'        = alpha' x0_hat + sqrt(1 - abar' - sigma_eta^2) eps
                     + sigma_eta z,
       z the full-image N(0, 1) draw of fast-grid index m (an INPUT here:
       synth/gen.py ddpm_noise); a stride-2 jump uses the same formula
       with t' = t_{m+2} and z_m.
  R34  second-order multistep solver (L66: "Lu et al. [31], [32] identified the
       semi-linear structure of diffusion ODEs and devised higher-order solvers"):
       the multistep DPM-Solver-2 of [31]/[32] in noise-prediction form, i.e. Eq. 3
       with eps replaced by
         D = eps_s + (eps_s - eps_prev) / (2 r),   r = h_prev / h,
       h = lambda_{t'} - lambda_s, h_prev = lambda_s - lambda_{s_prev}, where
       (eps_prev, s_prev) are the eps and timestep of the SAME band's previous
       step (a tier-2 rank's history spans its own stride); the first step of a
       band has no history and is Eq. 3 itself.
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


def ddpm_step(abar, x, eps, t, t_prev, z):
    """R19: eta = 1 step of [28] Eq. 12 from t to t_prev with noise z."""
    ab = abar[t]
    ab2 = abar[0] if t_prev < 0 else abar[t_prev]
    x0 = (x - np.sqrt(1.0 - ab) * eps) / np.sqrt(ab)
    s_eta = np.sqrt((1.0 - ab2) / (1.0 - ab)) * np.sqrt(1.0 - ab / ab2)
    return np.sqrt(ab2) * x0 + np.sqrt(1.0 - ab2 - s_eta ** 2) * eps + s_eta * z


def lam(abar, t):
    """lambda_t = log(alpha_t / sigma_t) (t = -1: alpha_bar_0, R18)."""
    return alpha_sigma(abar, t)[2]


def dpm2m_step(abar, x, eps, t, t_prev, hist):
    """R34: multistep DPM-Solver-2 (noise prediction) from t to t_prev.  hist =
    None (first step: Eq. 3) or (eps_prev, s_prev): the previous step of this band
    went s_prev -> t with eps_prev."""
    A, Bc = ddim_coeffs(abar, t, t_prev)
    if hist is None:
        return A * x + Bc * eps
    eps_p, s_prev = hist
    h = lam(abar, t_prev) - lam(abar, t)
    r = (lam(abar, t) - lam(abar, s_prev)) / h
    return A * x + Bc * (eps + (eps - eps_p) / (2.0 * r))


def cfg_combine(eps_u, eps_c, w):
    """R20: eps = eps_u + w (eps_c - eps_u)."""
    return eps_u + w * (eps_c - eps_u)
