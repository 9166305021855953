"""Oracle U-Net-family noise predictor eps_theta (float64 numpy), whole-image
and patch (row-band) forward with the stale-exchange sites.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's eps_theta is "U-Net [29] or DiTs [4]" and its
experiments use SDXL (L251-253, "a mix of convolutions and attention layers").
BASELINE.json C3 / C4 ask for SD-1.5- and SDXL-shaped U-Nets.  Weights are
random (R22), so only the *architecture* matters; it follows the diffusers
``UNet2DConditionModel`` layer list, written out plainly:

  time:   sinusoid(C0) [cos | sin] -> Linear(C0, 4C0) -> SiLU -> Linear(4C0, 4C0)
          (SDXL: + Linear/SiLU/Linear of [sinusoid256(time_ids) | pooled text])
  conv_in 3x3 (4 -> C0)
  down:   per level: n_res x [ResBlock (+ Transformer2D)] (+ Downsample, conv 3x3 s2)
  mid:    ResBlock, Transformer2D, ResBlock
  up:     per level: (n_res+1) x [concat skip -> ResBlock (+ Transformer2D)]
          (+ Upsample: nearest x2 -> conv 3x3)
  out:    GroupNorm -> SiLU -> conv 3x3 (C0 -> 4)
  ResBlock(x):   h = conv3x3(SiLU(GN(x))) + Linear(SiLU(temb));
                 h = conv3x3(SiLU(GN(h)));   out = skip(x) + h  (skip: 1x1 conv if C changes)
  Transformer2D: GN (eps 1e-6) -> proj_in -> depth x [x += SelfAttn(LN x);
                 x += CrossAttn(LN x, text); x += FF_GEGLU(LN x)] -> proj_out -> + input
                 (q/k/v without bias; out projections with bias; LN eps 1e-5, affine;
                 GEGLU: Linear(C, 8C) -> a * GELU_erf(g) -> Linear(4C, C))
  GroupNorm: 32 groups, affine; eps 1e-5 (ResBlocks, out) / 1e-6 (Transformer2D).

Patch parallelism (PAPER.md L80 / L171 "DistriFusion ... reuse stale
activations"): a rank owns latent rows [r0, r1) and runs every layer on its
band.  The band forward is a *generator*: at every exchange site it yields
``(kind, payload)`` and receives the assembled result from the caller, which
serves the rank's own FRESH payload plus the other ranks' payloads of the read
version (R14-R17).  Site kinds:

  "kv"   self-attention: payload (k, v) [B, n, d] of the band's tokens; result =
         the full-image (K, V) in row order (attention over own Q x full K/V).
  "halo" 3x3 conv input: payload (first, last) boundary rows of the band's conv
         input [B, 1, W, C]; result = (row above, row below) from the neighbour
         ranks (zeros at the image edge).  Stride-2 convs use only the row above;
         Upsample exchanges the PRE-upsample rows (R16); conv_in is an ordinary
         site (R15).
  "gn"   GroupNorm: payload (S1, S2, n) partial sums per (b, group) of the band;
         result = the sums over all ranks; mean = S1/n, var = max(S2/n - mean^2, 0)
         (R17).
Everything else (linear, 1x1 conv, LayerNorm, cross-attention) is band-local.
"""
from __future__ import annotations

import math

import numpy as np

# The layer list / channel bookkeeping is the architecture DESCRIPTION shared with
# the weight generator (synth/configs.py); it holds no arithmetic of the method.
from synth.configs import unet_levels as levels
from synth.configs import unet_up_io as up_resnet_io

from .dit import attention, linear, silu

GN_GROUPS = 32


# ----------------------------------------------------------------- primitives
def gelu_erf(x):
    """GELU(x) = x * Phi(x) (exact, erf form), the GEGLU activation."""
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def layernorm_affine(x, w, b, eps=1e-5):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * w + b


def conv3x3_valid(xp, w, b, stride=1):
    """Cross-correlation of an already padded NHWC input xp [B, Hp, Wp, Cin]
    with w [Cout, Cin, 3, 3] (PyTorch Conv2d layout), no further padding:
    out[b, y, x, o] = b[o] + sum_{c,ky,kx} xp[b, s*y+ky, s*x+kx, c] w[o, c, ky, kx]."""
    B, Hp, Wp, Cin = xp.shape
    Ho = (Hp - 3) // stride + 1
    Wo = (Wp - 3) // stride + 1
    out = np.zeros((B * Ho * Wo, w.shape[0]))
    for ky in range(3):
        for kx in range(3):
            patch = xp[:, ky:ky + stride * (Ho - 1) + 1:stride, kx:kx + stride * (Wo - 1) + 1:stride]
            # contiguous [pixels, Cin] x [Cin, Cout] operands: one BLAS product per tap
            out += np.ascontiguousarray(patch).reshape(-1, Cin) @ np.ascontiguousarray(w[:, :, ky, kx].T)
    return out.reshape(B, Ho, Wo, w.shape[0]) + b


def pad_cols(x):
    """Zero-pad one column left and right (the image's own left/right edges)."""
    return np.pad(x, ((0, 0), (0, 0), (1, 1), (0, 0)))


def gn_partials(x, groups=GN_GROUPS):
    """(S1, S2, n) per (batch, group) over the band x [B, h, W, C]."""
    B, h, W, C = x.shape
    g = x.reshape(B, h * W, groups, C // groups)
    s1 = g.sum(axis=(1, 3))
    s2 = (g * g).sum(axis=(1, 3))
    n = np.full((B, groups), float(h * W * (C // groups)))
    return s1, s2, n


def gn_apply(x, stats, w, b, eps, groups=GN_GROUPS):
    """Normalise x [B, h, W, C] with global (S1, S2, n): mean = S1/n,
    var = max(S2/n - mean^2, 0) (R17), then the per-channel affine."""
    s1, s2, n = stats
    mean = s1 / n
    var = np.maximum(s2 / n - mean * mean, 0.0)
    B, h, W, C = x.shape
    cg = C // groups
    m = np.repeat(mean, cg, axis=1)[:, None, None, :]
    v = np.repeat(var, cg, axis=1)[:, None, None, :]
    return (x - m) / np.sqrt(v + eps) * w + b


def group_norm_full(x, w, b, eps, groups=GN_GROUPS):
    """Textbook GroupNorm over the whole image (for pins)."""
    B, H, W, C = x.shape
    g = x.reshape(B, H * W, groups, C // groups)
    mu = g.mean(axis=(1, 3), keepdims=True)
    var = g.var(axis=(1, 3), keepdims=True)
    return ((g - mu) / np.sqrt(var + eps)).reshape(B, H, W, C) * w + b


def timestep_sinusoid(t, dim):
    """diffusers Timesteps(dim, flip_sin_to_cos=True, downscale_freq_shift=0):
    f_k = exp(-ln(10000) k / (dim/2)); emb = [cos(t f) | sin(t f)]."""
    half = dim // 2
    f = np.exp(-math.log(10000.0) * np.arange(half, dtype=np.float64) / half)
    a = np.asarray(t, dtype=np.float64)[..., None] * f
    return np.concatenate([np.cos(a), np.sin(a)], axis=-1)


# ----------------------------------------------------------------- the model
class UNet:
    def __init__(self, cfg: dict, weights: dict):
        self.cfg = cfg
        self.W = {k: np.asarray(v, dtype=np.float64) for k, v in weights.items()}
        self.L = levels(cfg)
        self.nres = cfg["layers_per_block"]

    # -- conditioning (per request / per timestep) ---------------------------
    def temb(self, t, cond):
        """Time embedding [B, 4 C0] (SDXL: + the micro-conditioning embedding)."""
        W, cfg = self.W, self.cfg
        B = cond["text"].shape[0]
        e = linear(silu(linear(timestep_sinusoid(t, cfg["channels"][0]), W["time.w1"],
                               W["time.b1"])), W["time.w2"], W["time.b2"])
        e = np.broadcast_to(e, (B, e.shape[-1])).copy()
        if cfg.get("add_embed"):
            tid = timestep_sinusoid(np.asarray(cond["time_ids"], dtype=np.float64), 256)
            a = np.concatenate([cond["pooled"], tid.reshape(B, -1)], axis=-1)
            e = e + linear(silu(linear(a, W["add.w1"], W["add.b1"])), W["add.w2"], W["add.b2"])
        return e

    # -- band-local building blocks (generators: yield exchange requests) ------
    def _gn(self, x, p, eps, act):
        stats = yield ("gn", gn_partials(x))
        y = gn_apply(x, stats, self.W[p + ".w"], self.W[p + ".b"], eps)
        return silu(y) if act else y

    def _conv(self, x, p, stride=1, upsample=False):
        """3x3 conv (pad 1) on the band x [B, h, W, C] with halo rows from the
        neighbours (zeros at the image's top / bottom edge)."""
        above, below = yield ("halo", (x[:, :1], x[:, -1:]))
        if upsample:  # nearest x2 of band + halos (R16: halos are pre-upsample rows)
            x = x.repeat(2, axis=1).repeat(2, axis=2)
            above = above.repeat(2, axis=2)
            below = below.repeat(2, axis=2)
        xp = np.concatenate([above, x, below], axis=1)
        if stride == 2:
            xp = xp[:, :-1]  # output row o reads input rows 2o-1 .. 2o+1 (top halo only)
        return conv3x3_valid(pad_cols(xp), self.W[p + ".w"], self.W[p + ".b"], stride)

    def _res(self, x, p, temb):
        W = self.W
        h = yield from self._gn(x, p + "norm1", 1e-5, True)
        h = yield from self._conv(h, p + "conv1")
        h = h + linear(silu(temb), W[p + "temb.w"], W[p + "temb.b"])[:, None, None, :]
        h = yield from self._gn(h, p + "norm2", 1e-5, True)
        h = yield from self._conv(h, p + "conv2")
        skip = x if (p + "skip.w") not in W else linear(x, W[p + "skip.w"], W[p + "skip.b"])
        return skip + h

    def _tr(self, x, p, depth, heads, text):
        W = self.W
        B, h, w, c = x.shape
        y = yield from self._gn(x, p + "norm", 1e-6, False)
        y = linear(y.reshape(B, h * w, c), W[p + "proj_in.w"], W[p + "proj_in.b"])
        for k in range(depth):
            q = f"{p}blk{k}."
            n1 = layernorm_affine(y, W[q + "ln1.w"], W[q + "ln1.b"])
            qq = n1 @ W[q + "attn1.q"].T
            kk = n1 @ W[q + "attn1.k"].T
            vv = n1 @ W[q + "attn1.v"].T
            kf, vf = yield ("kv", (kk, vv))
            y = y + linear(attention(qq, kf, vf, heads), W[q + "attn1.o"], W[q + "attn1.ob"])
            n2 = layernorm_affine(y, W[q + "ln2.w"], W[q + "ln2.b"])
            a2 = attention(n2 @ W[q + "attn2.q"].T, text @ W[q + "attn2.k"].T,
                           text @ W[q + "attn2.v"].T, heads)
            y = y + linear(a2, W[q + "attn2.o"], W[q + "attn2.ob"])
            n3 = layernorm_affine(y, W[q + "ln3.w"], W[q + "ln3.b"])
            f = linear(n3, W[q + "ff1.w"], W[q + "ff1.b"])
            a, g = f[..., :4 * c], f[..., 4 * c:]
            y = y + linear(a * gelu_erf(g), W[q + "ff2.w"], W[q + "ff2.b"])
        y = linear(y, W[p + "proj_out.w"], W[p + "proj_out.b"]).reshape(B, h, w, c)
        return x + y

    def band_forward(self, x_band, t, cond):
        """Generator: eps_theta on a latent band [h, W, C_in] -> [B, h, W, C_out]
        (h = band rows; the caller answers every exchange request)."""
        cfg, W = self.cfg, self.W
        B = cond["text"].shape[0]
        text = cond["text"]
        temb = self.temb(t, cond)
        x = np.broadcast_to(x_band.astype(np.float64), (B,) + x_band.shape).copy()
        h = yield from self._conv(x, "conv_in")
        skips = [h]
        for i, (c, att, depth, heads) in enumerate(self.L):
            for j in range(self.nres):
                h = yield from self._res(h, f"down{i}.res{j}.", temb)
                if att:
                    h = yield from self._tr(h, f"down{i}.attn{j}.", depth, heads, text)
                skips.append(h)
            if i < len(self.L) - 1:
                h = yield from self._conv(h, f"down{i}.ds", stride=2)
                skips.append(h)
        cm, _, _, hm = self.L[-1]
        h = yield from self._res(h, "mid.res0.", temb)
        h = yield from self._tr(h, "mid.attn.", cfg["mid_depth"], hm, text)
        h = yield from self._res(h, "mid.res1.", temb)
        rl = list(reversed(self.L))
        for i, lv in enumerate(up_resnet_io(cfg)):
            c, att, depth, heads = rl[i]
            for j in range(len(lv)):
                h = np.concatenate([h, skips.pop()], axis=-1)
                h = yield from self._res(h, f"up{i}.res{j}.", temb)
                if att:
                    h = yield from self._tr(h, f"up{i}.attn{j}.", depth, heads, text)
            if i < len(self.L) - 1:
                h = yield from self._conv(h, f"up{i}.us", upsample=True)
        h = yield from self._gn(h, "out.norm", 1e-5, True)
        return (yield from self._conv(h, "out.conv"))

    # -- unpatched forward ------------------------------------------------------
    def forward_full(self, x, t, cond):
        """eps_theta on the whole latent [H, W, C] -> [B, H, W, C] (one band,
        every exchange answered with the band's own data; image-edge halos 0)."""
        gen = self.band_forward(x, t, cond)
        return drive_single(gen)


def answer_alone(kind, payload):
    """Exchange answer for a single band covering the whole image."""
    if kind == "kv":
        return payload
    if kind == "halo":
        first, last = payload
        return np.zeros_like(first), np.zeros_like(last)
    if kind == "gn":
        return payload
    raise ValueError(kind)


def drive_single(gen):
    try:
        req = next(gen)
        while True:
            req = gen.send(answer_alone(*req))
    except StopIteration as e:
        return e.value


def guided_eps(cfg, eps_b):
    """R20: CFG combine of the internal batch (uncond, cond)."""
    w = cfg["guidance"]
    return eps_b[0] + w * (eps_b[1] - eps_b[0])
