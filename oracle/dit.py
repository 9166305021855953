"""Oracle DiT-family noise predictor eps_theta (float64 numpy).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's eps_theta(x, t) is "U-Net [29] or DiTs [4]"; its
experiments use SDXL (L253) and BASELINE.json adds DiT-XL/2 and PixArt-alpha
shapes.  Weights are random (R22), so only the *architecture* matters; it is
written out here plainly from SURVEY.md §8(c) O4 (DiT: Peebles & Xie, ref [4]):

  patchify (p=2, flatten order (c, dy, dx)) -> Linear(p^2 C_in -> d)
     + fixed 2-D sin-cos positional embedding of the token's global position
  t-embedding: sinusoid(256) -> Linear -> SiLU -> Linear
  class cond (DiT):  c = t_emb + y_table[label];   adaLN 6-way from SiLU(c)
  text cond (PixArt): adaLN-single  mod_l = sst_l + Linear(SiLU(t_emb)),
                      caption MLP 4096 -> d (GELU-tanh) -> d, cross-attention
  block:  h  = x + g1 * Attn(LN(x)(1+s1)+b1)
          h  = h + CrossAttn(h, y)                       (PixArt only)
          x' = h + g2 * MLP(LN(h)(1+s2)+b2)               MLP: 4d, GELU-tanh
  final:  Linear(LN(x)(1+s)+b) -> unpatchify, eps = first C_in channels
LayerNorm eps 1e-6, no affine.  Attention softmax(QK^T/sqrt(hd))V with biases.

Patch parallelism (DistriFusion ref [12]):
a band's tokens are its own queries; the keys/values it attends over are
supplied by the caller (own fresh rows + other ranks' rows of a given
version).  Every other op is band-local.  ``block_qkv`` / ``block_rest`` split
a block at that exchange site.

Activation layout here: [B, n_tokens, d] (tokens row-major over the band).
"""
from __future__ import annotations

import numpy as np

LN_EPS = 1e-6


# ----------------------------------------------------------------- primitives
def silu(x):
    return x / (1.0 + np.exp(-x))


def gelu_tanh(x):
    return 0.5 * x * (1.0 + np.tanh(np.sqrt(2.0 / np.pi) * (x + 0.044715 * x ** 3)))


def layernorm(x):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + LN_EPS)


def linear(x, w, b):
    """nn.Linear with weight [out, in]."""
    return x @ w.T + b


def attention(q, k, v, heads, q_chunk=1024):
    """softmax(q k^T / sqrt(hd)) v per head.  q [B,n,d], k/v [B,N,d].

    Every query row's softmax is independent of the others, so rows are
    evaluated in chunks of q_chunk (a memory bound for the full-resolution
    parity refs: 16384 x 16384 scores per head would not fit); the arithmetic of
    each row is the definition above, whatever the chunking."""
    B, n, d = q.shape
    if n > q_chunk:
        return np.concatenate([attention(q[:, i:i + q_chunk], k, v, heads, q_chunk)
                               for i in range(0, n, q_chunk)], axis=1)
    N = k.shape[1]
    hd = d // heads
    qh = q.reshape(B, n, heads, hd).transpose(0, 2, 1, 3)
    kh = k.reshape(B, N, heads, hd).transpose(0, 2, 1, 3)
    vh = v.reshape(B, N, heads, hd).transpose(0, 2, 1, 3)
    s = qh @ kh.transpose(0, 1, 3, 2) / np.sqrt(hd)
    s = s - s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p = p / p.sum(axis=-1, keepdims=True)
    o = p @ vh
    return o.transpose(0, 2, 1, 3).reshape(B, n, d)


def timestep_freq(t, dim=256, max_period=10000.0):
    """Sinusoidal timestep features [cos(t f_k), sin(t f_k)], f_k =
    exp(-ln(max_period) k / (dim/2)) (DiT ref [4] TimestepEmbedder)."""
    half = dim // 2
    f = np.exp(-np.log(max_period) * np.arange(half, dtype=np.float64) / half)
    a = float(t) * f
    return np.concatenate([np.cos(a), np.sin(a)])


def pos_embed(d, hp, wp):
    """Fixed 2-D sin-cos embedding of the full token grid [hp*wp, d]:
    [sin(c w), cos(c w), sin(r w), cos(r w)], w_k = 10000^(-k/(d/4))."""
    q = d // 4
    w = 1.0 / 10000.0 ** (np.arange(q, dtype=np.float64) / q)
    r, c = np.meshgrid(np.arange(hp, dtype=np.float64), np.arange(wp, dtype=np.float64),
                       indexing="ij")
    r = r.reshape(-1, 1) * w
    c = c.reshape(-1, 1) * w
    return np.concatenate([np.sin(c), np.cos(c), np.sin(r), np.cos(r)], axis=1)


# ----------------------------------------------------------------- the model
class DiT:
    def __init__(self, cfg: dict, weights: dict):
        self.cfg = cfg
        self.W = {k: np.asarray(v, dtype=np.float64) for k, v in weights.items()}
        self.d = cfg["hidden"]
        self.H = cfg["heads"]
        self.p = cfg["patch"]
        self.depth = cfg["depth"]
        self.hp = cfg["latent_h"] // self.p
        self.wp = cfg["latent_w"] // self.p
        self.pos = pos_embed(self.d, self.hp, self.wp)
        self.text = cfg["cond"] == "text"

    # -- conditioning (per request, per timestep) -----------------------------
    def caption(self, cond):
        """PixArt caption projection y = W2 GELU_tanh(W1 text + b1) + b2."""
        if not self.text:
            return None
        W = self.W
        return linear(gelu_tanh(linear(cond["text"], W["caption.w1"], W["caption.b1"])),
                      W["caption.w2"], W["caption.b2"])

    def modulations(self, t, cond):
        """Per-block (shift1, scale1, gate1, shift2, scale2, gate2) [B, d] each
        and final (shift, scale)."""
        W, d = self.W, self.d
        temb = linear(silu(linear(timestep_freq(t), W["t_embed.w1"], W["t_embed.b1"])),
                      W["t_embed.w2"], W["t_embed.b2"])
        mods = []
        if self.text:
            B = cond["text"].shape[0]
            t0 = linear(silu(temb), W["t_block.w"], W["t_block.b"])           # [6d]
            for l in range(self.depth):
                m = W[f"blocks.{l}.sst"].reshape(-1) + t0
                mods.append(np.broadcast_to(m, (B, 6 * d)).reshape(B, 6, d))
            sst = W["final.sst"]
            fin = np.stack([sst[0] + temb, sst[1] + temb])[None].repeat(B, 0)  # [B,2,d]
        else:
            c = temb[None, :] + W["y_embed.table"][cond["labels"]]            # [B, d]
            sc = silu(c)
            for l in range(self.depth):
                mods.append(linear(sc, W[f"blocks.{l}.ada.w"], W[f"blocks.{l}.ada.b"])
                            .reshape(-1, 6, d))
            fin = linear(sc, W["final.ada.w"], W["final.ada.b"]).reshape(-1, 2, d)
        return mods, fin

    # -- band-local pieces ---------------------------------------------------
    def embed(self, x_band, tok_row0, B):
        """Patchify a latent band [rows, W, C] (rows = multiple of p) whose first
        token row is global token row tok_row0 -> [B, n, d]."""
        p, d = self.p, self.d
        rows, wlat, C = x_band.shape
        hr, wc = rows // p, wlat // p
        patches = (x_band.reshape(hr, p, wc, p, C).transpose(0, 2, 4, 1, 3)
                   .reshape(hr * wc, C * p * p))                      # column = c*p*p + dy*p + dx
        tok = linear(patches, self.W["x_embed.w"], self.W["x_embed.b"])
        tok = tok + self.pos[tok_row0 * self.wp:(tok_row0 + hr) * self.wp]
        return np.broadcast_to(tok, (B,) + tok.shape).copy()

    def block_qkv(self, l, h, mod):
        """Self-attention site inputs: (q, k, v) of the band's own tokens."""
        W = self.W
        x = layernorm(h) * (1.0 + mod[:, 1][:, None]) + mod[:, 0][:, None]
        qkv = linear(x, W[f"blocks.{l}.qkv.w"], W[f"blocks.{l}.qkv.b"])
        d = self.d
        return qkv[..., :d], qkv[..., d:2 * d], qkv[..., 2 * d:]

    def block_rest(self, l, h, q, k_full, v_full, mod, y):
        """Everything of block l after the exchange site."""
        W = self.W
        a = attention(q, k_full, v_full, self.H)
        h = h + mod[:, 2][:, None] * linear(a, W[f"blocks.{l}.proj.w"], W[f"blocks.{l}.proj.b"])
        if self.text:
            d = self.d
            xq = linear(h, W[f"blocks.{l}.xq.w"], W[f"blocks.{l}.xq.b"])
            kv = linear(y, W[f"blocks.{l}.xkv.w"], W[f"blocks.{l}.xkv.b"])
            xa = attention(xq, kv[..., :d], kv[..., d:], self.H)
            h = h + linear(xa, W[f"blocks.{l}.xproj.w"], W[f"blocks.{l}.xproj.b"])
        x = layernorm(h) * (1.0 + mod[:, 4][:, None]) + mod[:, 3][:, None]
        m = linear(gelu_tanh(linear(x, W[f"blocks.{l}.fc1.w"], W[f"blocks.{l}.fc1.b"])),
                   W[f"blocks.{l}.fc2.w"], W[f"blocks.{l}.fc2.b"])
        return h + mod[:, 5][:, None] * m

    def final(self, h, fin, rows):
        """Final adaLN + linear + unpatchify -> eps [B, rows, W, C_in]."""
        p, C = self.p, self.cfg["c_out"]
        x = layernorm(h) * (1.0 + fin[:, 1][:, None]) + fin[:, 0][:, None]
        o = linear(x, self.W["final.linear.w"], self.W["final.linear.b"])   # [B, n, p*p*C]
        B = o.shape[0]
        hr, wc = rows // p, self.wp
        img = o.reshape(B, hr, wc, p, p, C).transpose(0, 1, 3, 2, 4, 5).reshape(B, rows, wc * p, C)
        return img[..., :self.cfg["c_in"]]

    # -- unpatched forward (the "no patch parallelism" reference) -------------
    def forward_full(self, x, t, cond, y=None):
        """eps_theta(x, t) on the full latent [H, W, C] -> [B, H, W, C]."""
        B = batch_of(self.cfg)
        if y is None:
            y = self.caption(cond)
        mods, fin = self.modulations(t, cond)
        h = self.embed(x, 0, B)
        for l in range(self.depth):
            q, k, v = self.block_qkv(l, h, mods[l])
            h = self.block_rest(l, h, q, k, v, mods[l], y)
        return self.final(h, fin, x.shape[0])


def batch_of(cfg):
    return 2 if cfg.get("guidance") else 1


def guided_eps(cfg, eps_b):
    """R20: combine the internal batch into one eps [rows, W, C]."""
    if eps_b.shape[0] == 1:
        return eps_b[0]
    w = cfg["guidance"]
    return eps_b[0] + w * (eps_b[1] - eps_b[0])
