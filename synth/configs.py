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
    # tiny U-Net for fast oracle pins / parity (2 levels, SDXL-style add embedding)
    "tiny_unet": dict(
        family="unet", cond="text", channels=[64, 128], tdepth=[0, 1], mid_depth=1,
        heads=None, head_dim=16, layers_per_block=1, c_in=4, c_out=4,
        latent_h=16, latent_w=16, text_len=8, text_dim=64, add_embed=True,
        pooled_dim=64, time_ids=[64, 64, 0, 0, 64, 64], guidance=5.0,
        schedule="scaled_linear",
    ),
    # C3: SD-1.5 shaped U-Net, 512^2 image -> 64x64 latent, CLIP-L text 77x768
    "sd15": dict(
        family="unet", cond="text", channels=[320, 640, 1280, 1280], tdepth=[1, 1, 1, 0],
        mid_depth=1, heads=8, head_dim=None, layers_per_block=2, c_in=4, c_out=4,
        latent_h=64, latent_w=64, text_len=77, text_dim=768, add_embed=False,
        guidance=7.5, schedule="scaled_linear",
    ),
    # C4: SDXL shaped U-Net, 1024^2 image -> 128x128 latent, text 77x2048 + pooled
    # 1280 + 6 micro-conditioning time ids
    "sdxl": dict(
        family="unet", cond="text", channels=[320, 640, 1280], tdepth=[0, 2, 10],
        mid_depth=10, heads=None, head_dim=64, layers_per_block=2, c_in=4, c_out=4,
        latent_h=128, latent_w=128, text_len=77, text_dim=2048, add_embed=True,
        pooled_dim=1280, time_ids=[1024, 1024, 0, 0, 1024, 1024],
        guidance=5.0, schedule="scaled_linear",
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
    "C3": dict(model="sd15", n_gpus=4, speeds=None, m_base=50, m_warmup=4,
               occupancy=[0, 20, 40, 60]),
    "C4": dict(model="sdxl", n_gpus=8, speeds=None, m_base=50, m_warmup=4,
               occupancy=[0, 0, 20, 20, 40, 40, 60, 60]),
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


def rows_per_unit(cfg: dict) -> int:
    """Latent rows per planner unit: one row of the coarsest feature
    map — p for a DiT (one token row), 2^(levels-1) for a U-Net."""
    if cfg["family"] == "unet":
        return 2 ** (len(cfg["channels"]) - 1)
    return cfg["patch"]


def tokens_hw(cfg: dict) -> tuple[int, int]:
    p = cfg["patch"]
    return cfg["latent_h"] // p, cfg["latent_w"] // p


def manifest(cfg: dict) -> list[tuple[str, tuple[int, ...], str]]:
    """Weight tensors of a model preset in load order (DiT or U-Net family)."""
    if cfg["family"] == "unet":
        return unet_manifest(cfg)
    return dit_manifest(cfg)


def dit_manifest(cfg: dict) -> list[tuple[str, tuple[int, ...], str]]:
    """DiT-family weight tensors in load order: (name, shape, init-kind).

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


# ---------------------------------------------------------------------------
# U-Net family architecture description (C3 SD-1.5, C4 SDXL shapes; diffusers
# UNet2DConditionModel layer list)
# ---------------------------------------------------------------------------
def unet_levels(cfg):
    """Per level: (channels, has_attention, transformer depth, heads)."""
    out = []
    for i, c in enumerate(cfg["channels"]):
        depth = cfg["tdepth"][i]
        heads = c // cfg["head_dim"] if cfg.get("head_dim") else cfg["heads"]
        out.append((c, depth > 0, depth, heads))
    return out


def unet_up_io(cfg):
    """diffusers' channel bookkeeping of the up path: list per up level of
    [(in_ch, skip_ch, out_ch)] for its n_res+1 ResBlocks (skips popped from
    the end of the down-path stack)."""
    ch = cfg["channels"]
    nres = cfg["layers_per_block"]
    rev = list(reversed(ch))
    res = []
    prev = rev[0]
    for i, oc in enumerate(rev):
        ic = rev[min(i + 1, len(ch) - 1)]
        lv = []
        for j in range(nres + 1):
            skip = ic if j == nres else oc
            rin = prev if j == 0 else oc
            lv.append((rin, skip, oc))
        res.append(lv)
        prev = oc
    return res


def unet_manifest(cfg):
    """Weight tensors in load order: (name, shape, init-kind).  Conv weights are
    [Cout, Cin, 3, 3] / [Cout, Cin] (1x1), linear weights [out, in].  init-kind
    as synth/configs.manifest: 'w' N(0, 1/fan_in), 'wo' residual-branch output
    N(0, 1/fan_in)/sqrt(2 n_blocks), 'b' N(0, 0.02^2), 'g' GN/LN gain
    1 + N(0, 0.02^2)."""
    C0 = cfg["channels"][0]
    td = 4 * C0
    L = unet_levels(cfg)
    m = []

    def res(p, cin, cout):
        m.extend([(p + "norm1.w", (cin,), "g"), (p + "norm1.b", (cin,), "b"),
                  (p + "conv1.w", (cout, cin, 3, 3), "w"), (p + "conv1.b", (cout,), "b"),
                  (p + "temb.w", (cout, td), "w"), (p + "temb.b", (cout,), "b"),
                  (p + "norm2.w", (cout,), "g"), (p + "norm2.b", (cout,), "b"),
                  (p + "conv2.w", (cout, cout, 3, 3), "wo"), (p + "conv2.b", (cout,), "b")])
        if cin != cout:
            m.extend([(p + "skip.w", (cout, cin), "w"), (p + "skip.b", (cout,), "b")])

    def tr(p, c, depth):
        ctx = cfg["text_dim"]
        m.extend([(p + "norm.w", (c,), "g"), (p + "norm.b", (c,), "b"),
                  (p + "proj_in.w", (c, c), "w"), (p + "proj_in.b", (c,), "b")])
        for k in range(depth):
            q = f"{p}blk{k}."
            m.extend([(q + "ln1.w", (c,), "g"), (q + "ln1.b", (c,), "b"),
                      (q + "attn1.q", (c, c), "w"), (q + "attn1.k", (c, c), "w"),
                      (q + "attn1.v", (c, c), "w"), (q + "attn1.o", (c, c), "wo"),
                      (q + "attn1.ob", (c,), "b"),
                      (q + "ln2.w", (c,), "g"), (q + "ln2.b", (c,), "b"),
                      (q + "attn2.q", (c, c), "w"), (q + "attn2.k", (c, ctx), "w"),
                      (q + "attn2.v", (c, ctx), "w"), (q + "attn2.o", (c, c), "wo"),
                      (q + "attn2.ob", (c,), "b"),
                      (q + "ln3.w", (c,), "g"), (q + "ln3.b", (c,), "b"),
                      (q + "ff1.w", (8 * c, c), "w"), (q + "ff1.b", (8 * c,), "b"),
                      (q + "ff2.w", (c, 4 * c), "wo"), (q + "ff2.b", (c,), "b")])
        m.extend([(p + "proj_out.w", (c, c), "wo"), (p + "proj_out.b", (c,), "b")])

    m.extend([("time.w1", (td, C0), "w"), ("time.b1", (td,), "b"),
              ("time.w2", (td, td), "w"), ("time.b2", (td,), "b")])
    if cfg.get("add_embed"):
        m.extend([("add.w1", (td, 6 * 256 + cfg["pooled_dim"]), "w"), ("add.b1", (td,), "b"),
                  ("add.w2", (td, td), "w"), ("add.b2", (td,), "b")])
    m.extend([("conv_in.w", (C0, cfg["c_in"], 3, 3), "w"), ("conv_in.b", (C0,), "b")])
    prev = C0
    for i, (c, att, depth, _) in enumerate(L):
        for j in range(cfg["layers_per_block"]):
            res(f"down{i}.res{j}.", prev if j == 0 else c, c)
            if att:
                tr(f"down{i}.attn{j}.", c, depth)
        if i < len(L) - 1:
            m.extend([(f"down{i}.ds.w", (c, c, 3, 3), "w"), (f"down{i}.ds.b", (c,), "b")])
        prev = c
    cm, _, dmid, _ = L[-1]
    res("mid.res0.", cm, cm)
    tr("mid.attn.", cm, cfg["mid_depth"])
    res("mid.res1.", cm, cm)
    rl = list(reversed(L))
    for i, lv in enumerate(unet_up_io(cfg)):
        c, att, depth, _ = rl[i]
        for j, (rin, skip, oc) in enumerate(lv):
            res(f"up{i}.res{j}.", rin + skip, oc)
            if att:
                tr(f"up{i}.attn{j}.", oc, depth)
        if i < len(L) - 1:
            m.extend([(f"up{i}.us.w", (c, c, 3, 3), "w"), (f"up{i}.us.b", (c,), "b")])
    m.extend([("out.norm.w", (C0,), "g"), ("out.norm.b", (C0,), "b"),
              ("out.conv.w", (cfg["c_out"], C0, 3, 3), "w"), ("out.conv.b", (cfg["c_out"],), "b")])
    return m
