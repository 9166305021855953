"""Workload presets (BASELINE.json ``configs`` C1..C5; SURVEY.md §8(c) O4 shapes,
§8(d) "Concrete synthetic input").  Pure data: no method arithmetic.

Model presets describe random-init networks *shaped like* the paper's
workloads (PAPER.md L251-253 uses SDXL; BASELINE.json adds DiT / PixArt
shapes).  Run presets bind a model to a GPU count, occupancy pattern and the
STADI hyper-parameters of PAPER.md L284 (M_warmup = 4, a = 0.75, b = 0.25).
"""
from __future__ import annotations

import copy

# ---------------------------------------------------------------------------
# DiT-family model presets
# ---------------------------------------------------------------------------
MODELS = {
    # C1: "tiny DiT (2 blocks, hidden 64, 4 heads) on 16x16x4 latent"
    "tiny_dit": dict(
        family="dit", cond="class", hidden=64, heads=4, depth=2, patch=2,
        c_in=4, c_out=4, latent_h=16, latent_w=16, num_classes=10,
        class_label=3, guidance=None, schedule="linear",
    ),
    # C2: DiT-XL/2 shaped, 256^2 image -> 32x32 latent, class-conditional, CFG
    "dit_xl2": dict(
        family="dit", cond="class", hidden=1152, heads=16, depth=28, patch=2,
        c_in=4, c_out=8, latent_h=32, latent_w=32, num_classes=1000,
        class_label=207, guidance=4.0, schedule="linear",
    ),
    # C5: PixArt-alpha shaped, 2048^2 image -> 256x256 latent, T5 text (120x4096)
    "pixart_alpha": dict(
        family="dit", cond="text", hidden=1152, heads=16, depth=28, patch=2,
        c_in=4, c_out=8, latent_h=256, latent_w=256, text_len=120,
        text_dim=4096, guidance=4.5, schedule="linear",
    ),
}

# ---------------------------------------------------------------------------
# Run presets (BASELINE.json configs[0..4]).  speeds: given speeds (C1 only);
# occupancy: emulated background load per GPU in percent.
# ---------------------------------------------------------------------------
RUNS = {
    "C1": dict(model="tiny_dit", n_gpus=2, speeds=[1.0, 0.5], m_base=10,
               m_warmup=2, occupancy=None),
    "C2": dict(model="dit_xl2", n_gpus=2, speeds=None, m_base=50, m_warmup=4,
               occupancy=[0, 40]),
    "C5": dict(model="pixart_alpha", n_gpus=None, speeds=None, m_base=20,
               m_warmup=4, occupancy="half50"),
}

# STADI hyper-parameters, PAPER.md L284 (V-A "Implementation Details").
A_NUM, A_DEN = 3, 4      # a = 0.75
B_NUM, B_DEN = 1, 4      # b = 0.25

# Seeds, SURVEY §8(d) "Common inputs".
SEED_WEIGHTS = 0
SEED_NOISE = 1234
SEED_COND = 42


def model(name: str, **overrides) -> dict:
    """Return a copy of a model preset with optional overrides (e.g. depth=2,
    latent_h=64 for the depth/resolution-reduced parity variants)."""
    cfg = copy.deepcopy(MODELS[name])
    cfg.update(overrides)
    cfg["name"] = name
    return cfg


def batch(cfg: dict) -> int:
    """Internal batch B: 2 with classifier-free guidance (uncond, cond), else 1
    (SURVEY R20)."""
    return 2 if cfg.get("guidance") else 1


def tokens_hw(cfg: dict) -> tuple[int, int]:
    p = cfg["patch"]
    return cfg["latent_h"] // p, cfg["latent_w"] // p


def manifest(cfg: dict) -> list[tuple[str, tuple[int, ...], str]]:
    """Weight tensors in load order: (name, shape, init-kind).

    Linear weights are stored [out, in] (row = output feature).  init-kind is
    one of  'w' (N(0, 1/fan_in)), 'wo' (residual-branch output projection,
    N(0, 1/fan_in)/sqrt(2*depth)), 'b' (bias, N(0, 0.02^2)), 'emb'
    (class table, N(0, 0.5^2)), 'table' (PixArt scale-shift table,
    N(0,1)/sqrt(hidden)).  SURVEY §8(c) R22: NOT adaLN-Zero.
    The same order is documented in include/stadi.h (stadi_load_weights).
    """
    d = cfg["hidden"]
    p = cfg["patch"]
    L = cfg["depth"]
    text = cfg["cond"] == "text"
    m: list[tuple[str, tuple[int, ...], str]] = []
    m += [("x_embed.w", (d, cfg["c_in"] * p * p), "w"), ("x_embed.b", (d,), "b")]
    m += [("t_embed.w1", (d, 256), "w"), ("t_embed.b1", (d,), "b"),
          ("t_embed.w2", (d, d), "w"), ("t_embed.b2", (d,), "b")]
    if text:
        m += [("t_block.w", (6 * d, d), "w"), ("t_block.b", (6 * d,), "b"),
              ("caption.w1", (d, cfg["text_dim"]), "w"), ("caption.b1", (d,), "b"),
              ("caption.w2", (d, d), "w"), ("caption.b2", (d,), "b")]
    else:
        m += [("y_embed.table", (cfg["num_classes"] + 1, d), "emb")]
    for l in range(L):
        pre = f"blocks.{l}."
        if text:
            m += [(pre + "sst", (6, d), "table")]
        else:
            m += [(pre + "ada.w", (6 * d, d), "w"), (pre + "ada.b", (6 * d,), "b")]
        m += [(pre + "qkv.w", (3 * d, d), "w"), (pre + "qkv.b", (3 * d,), "b"),
              (pre + "proj.w", (d, d), "wo"), (pre + "proj.b", (d,), "b")]
        if text:
            m += [(pre + "xq.w", (d, d), "w"), (pre + "xq.b", (d,), "b"),
                  (pre + "xkv.w", (2 * d, d), "w"), (pre + "xkv.b", (2 * d,), "b"),
                  (pre + "xproj.w", (d, d), "wo"), (pre + "xproj.b", (d,), "b")]
        m += [(pre + "fc1.w", (4 * d, d), "w"), (pre + "fc1.b", (4 * d,), "b"),
              (pre + "fc2.w", (d, 4 * d), "wo"), (pre + "fc2.b", (d,), "b")]
    if text:
        m += [("final.sst", (2, d), "table")]
    else:
        m += [("final.ada.w", (2 * d, d), "w"), ("final.ada.b", (2 * d,), "b")]
    m += [("final.linear.w", (p * p * cfg["c_out"], d), "w"),
          ("final.linear.b", (p * p * cfg["c_out"],), "b")]
    return m
