"""Seeded input generators (numpy PCG64).  No method arithmetic here.

SURVEY.md §8(d) "Common inputs": noise ~ N(0,1) fp32 (seed 1234), weights
seed 0, conditioning seed 42.  R22: random init, not adaLN-Zero.
"""
from __future__ import annotations

import numpy as np

from . import configs


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def weights(cfg: dict, seed: int = configs.SEED_WEIGHTS) -> dict[str, np.ndarray]:
    """Random-init weights in manifest order (float32, C-contiguous).

    fan_in = the input features of a linear / 1x1 conv ([out, in]) or
    in_channels * 9 of a 3x3 conv ([out, in, 3, 3]).  The residual-branch
    scaling uses the number of residual blocks: depth (DiT) or the number of
    'wo' tensors / 2 (U-Net: ResBlock conv2 + attention / FF outputs)."""
    rng = _rng(seed)
    man = configs.manifest(cfg)
    if cfg["family"] == "unet":
        nblk = max(1, sum(1 for _, _, k in man if k == "wo") // 2)
    else:
        nblk = cfg["depth"]
    out: dict[str, np.ndarray] = {}
    for name, shape, kind in man:
        a = rng.standard_normal(shape, dtype=np.float32)
        fan_in = int(np.prod(shape[1:])) if len(shape) > 1 else 1
        if kind == "w":
            a *= np.float32(1.0 / np.sqrt(fan_in))
        elif kind == "wo":
            a *= np.float32(1.0 / np.sqrt(fan_in) / np.sqrt(2.0 * nblk))
        elif kind == "b":
            a *= np.float32(0.02)
        elif kind == "g":
            a = np.float32(1.0) + a * np.float32(0.02)
        elif kind == "emb":
            a *= np.float32(0.5)
        elif kind == "table":
            a *= np.float32(1.0 / np.sqrt(cfg["hidden"]))
        else:  # pragma: no cover
            raise ValueError(kind)
        out[name] = np.ascontiguousarray(a, dtype=np.float32)
    return out


def noise(cfg: dict, seed: int = configs.SEED_NOISE) -> np.ndarray:
    """Initial latent x_T: [H, W, C_in] float32 ~ N(0, 1) (NHWC, full image)."""
    return _rng(seed).standard_normal(
        (cfg["latent_h"], cfg["latent_w"], cfg["c_in"]), dtype=np.float32)


def cond(cfg: dict, seed: int = configs.SEED_COND) -> dict:
    """Conditioning for the internal batch (index 0 = unconditional when CFG).

    class-conditional: labels [B] (null class = num_classes for the uncond row).
    text-conditional:  text [B, L_txt, D_txt] float32 ~ N(0,1) (R21: synthetic
    T5 / CLIP-shaped embeddings; row 0 plays the null caption); SDXL adds
    pooled [B, 1280] ~ N(0,1) and the micro-conditioning time_ids [B, 6].
    """
    B = configs.batch(cfg)
    if cfg["cond"] == "class":
        lab = [cfg["class_label"]] if B == 1 else [cfg["num_classes"], cfg["class_label"]]
        return {"labels": np.asarray(lab, dtype=np.int32)}
    rng = _rng(seed)
    out = {"text": rng.standard_normal((B, cfg["text_len"], cfg["text_dim"]), dtype=np.float32)}
    if cfg.get("add_embed"):
        out["pooled"] = rng.standard_normal((B, cfg["pooled_dim"]), dtype=np.float32)
        out["time_ids"] = np.tile(np.asarray(cfg["time_ids"], dtype=np.float32), (B, 1))
    return out


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float32 -> bfloat16 (round-to-nearest-even), returned as float32.

    Input transform for bf16 parity runs (R22: the oracle consumes the same
    bf16-rounded weights the device stores).  NaN/Inf are not expected here.
    """
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(a.shape)


def weights_bf16(w: dict[str, np.ndarray]) -> dict[str, np.ndarray]:
    return {k: bf16_round(v) for k, v in w.items()}


# ------------------------------------------------------------------ DDPM noise
# R19: the DDPM (eta = 1) sampler adds sigma_eta * z_m, z_m a
# full-image N(0, 1) tensor per fast-grid index m.  Both sides implement the
# same counter-based generator (the CUDA sampler draws z in-kernel, the oracle
# receives it from here), so nothing has to be copied per step:
#   Philox4x64-10 (Salmon et al., SC'11; numpy's np.random.Philox), key =
#   (seed, m), counter = (e >> 2, 0, 0, 0) for the element with flat index e of
#   the full [H, W, C] image, 64-bit word = lane e & 3 of that block;
#   u1 = ((w >> 40) + 1/2) 2^-24, u2 = (((w >> 16) & (2^24 - 1)) + 1/2) 2^-24,
#   z = sqrt(-2 ln u1) cos(2 pi u2)            (Box-Muller, cosine branch).
# 24-bit uniforms are exact in fp32, so the device's fp32 transform differs
# from this fp64 one only by rounding (~1e-7 relative).
SEED_DDPM = 2024
_ALL_ONES = (1 << 64) - 1


def philox_words(seed: int, m: int, n_words: int) -> np.ndarray:
    """The first n_words 64-bit outputs of Philox4x64-10 with key (seed, m),
    counter blocks 0, 1, 2, ... (numpy increments the counter before each
    block, so it starts from all-ones = -1)."""
    g = np.random.Philox(counter=[_ALL_ONES] * 4, key=[seed & _ALL_ONES, m & _ALL_ONES])
    return g.random_raw(n_words)


def ddpm_noise(shape, m: int, seed: int = SEED_DDPM) -> np.ndarray:
    """z_m for fast-grid index m: full-image [H, W, C] float64 ~ N(0, 1)."""
    n = int(np.prod(shape))
    w = philox_words(seed, m, n).astype(np.uint64)
    u1 = ((w >> np.uint64(40)).astype(np.float64) + 0.5) * 2.0 ** -24
    u2 = (((w >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(np.float64) + 0.5) * 2.0 ** -24
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return z.reshape(shape)
