"""Pins of the U-Net oracle (oracle/unet.py) — CPU only.

What fixes the U-Net family independently of the oracle's own code:
* diffusers' published parameter counts of the SD-1.5 UNet (859,520,964) and the
  SDXL UNet (2,567,463,684) — an exact count pins every layer shape / channel
  bookkeeping of the architecture description (synth/configs.py);
* the up-path ResBlock input widths of SD-1.5 (its conv1 weight shapes);
* conv3x3 against a brute-force 7-deep loop; GroupNorm against a textbook
  formula; GELU(1) = Phi(1) = 0.8413447460685429; sinusoid closed forms;
* the whole layer composition against an independent per-element evaluation
  written from the diffusers layer definitions (test_unet_forward_bruteforce on
  a micro config that has every layer kind; mutating the oracle -- swapped skip
  concat, swapped GEGLU halves, GN eps 1e-6 -> 1e-5, LN eps 1e-5 -> 1e-6, a
  dropped Transformer2D residual, a sign flip of the add-embedding -- moves it
  by >= 4e-7 relative against a 1e-11 tolerance);
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
    # R32 odd K = 3: the slow GPU's stride is 3
    seq5 = OR.sequential(cfg, W, x, c, 5)
    p = OR.plan_for(cfg, [4, 2], 5, 2)
    assert p["sync_period"] == 3 and p["steps"] == [5, 3]
    out = OR.run(cfg, W, x, c, p)
    assert np.max(np.abs(out - seq5)) <= 1e-12 * np.max(np.abs(seq5))


# ----------------------------------------------------------- brute-force U-Net
def _micro_cfg():
    """Micro U-Net that still exercises every layer kind of the diffusers
    UNet2DConditionModel: 2 levels (channels 32 / 64, GroupNorm 32 groups),
    2 ResBlocks per down level (so the up path pops 3 skips per level, one
    from a Downsample), a 1x1 skip conv where channels change, Transformer2D
    (depth 1) on BOTH levels and in the mid block, Downsample / Upsample,
    SDXL add-embedding, CFG batch of 2."""
    return dict(family="unet", cond="text", channels=[32, 64], tdepth=[1, 1], mid_depth=1,
                heads=None, head_dim=16, layers_per_block=2, c_in=4, c_out=4, latent_h=8,
                latent_w=8, text_len=3, text_dim=8, add_embed=True, pooled_dim=8,
                time_ids=[16, 16, 0, 0, 16, 16], guidance=5.0, schedule="scaled_linear",
                name="micro_unet")


def _brute_unet(cfg, W, x, t, cond):
    """eps_theta of the U-Net family by per-element loops, written from the
    diffusers UNet2DConditionModel / ResnetBlock2D / Transformer2DModel /
    BasicTransformerBlock / GEGLU / Downsample2D / Upsample2D definitions
    (SURVEY §8(c) O4), independently of oracle/unet.py: matrix-vector products
    per pixel / token are the only library primitive.  Channel counts are read
    off the tensors (the up path's concat widths are not taken from the
    architecture description).  Returns [B, H, W, C_out]."""
    W = {k: np.asarray(v, np.float64) for k, v in W.items()}
    ch = cfg["channels"]
    nlev, nres = len(ch), cfg["layers_per_block"]
    B = 2 if cfg.get("guidance") else 1
    text = np.asarray(cond["text"], np.float64)

    def silu(v):
        return v / (1.0 + np.exp(-v))

    def sinusoid(tv, dim):                      # Timesteps(dim, flip_sin_to_cos=True, shift 0)
        half = dim // 2
        f = [math.exp(-math.log(10000.0) * k / half) for k in range(half)]
        return np.array([math.cos(tv * fk) for fk in f] + [math.sin(tv * fk) for fk in f])

    def mv(w, v, b=None):                       # Linear: y = W v (+ b)
        y = w @ v
        return y if b is None else y + b

    def conv(h, p, stride=1):                   # Conv2d(k=3, padding=1, stride)
        wt, bs = W[p + ".w"], W[p + ".b"]
        nb, H, Wd, _ = h.shape
        Ho, Wo = (H - 1) // stride + 1, (Wd - 1) // stride + 1
        out = np.zeros((nb, Ho, Wo, wt.shape[0]))
        for b in range(nb):
            for oy in range(Ho):
                for ox in range(Wo):
                    acc = bs.copy()
                    for ky in range(3):
                        iy = oy * stride + ky - 1
                        if not 0 <= iy < H:
                            continue
                        for kx in range(3):
                            ix = ox * stride + kx - 1
                            if 0 <= ix < Wd:
                                acc += wt[:, :, ky, kx] @ h[b, iy, ix]
                    out[b, oy, ox] = acc
        return out

    def groupnorm(h, p, eps):                   # GroupNorm(32, C, eps, affine)
        nb, H, Wd, C = h.shape
        cg = C // 32
        out = np.zeros_like(h)
        for b in range(nb):
            for g in range(32):
                vals = [h[b, y, xx, c] for y in range(H) for xx in range(Wd)
                        for c in range(g * cg, (g + 1) * cg)]
                mu = math.fsum(vals) / len(vals)
                var = math.fsum((v - mu) ** 2 for v in vals) / len(vals)
                for c in range(g * cg, (g + 1) * cg):
                    out[b, :, :, c] = (h[b, :, :, c] - mu) / math.sqrt(var + eps) \
                        * W[p + ".w"][c] + W[p + ".b"][c]
        return out

    def layernorm(v, p):                        # LayerNorm(C, eps 1e-5, affine)
        mu = math.fsum(v) / len(v)
        var = math.fsum((a - mu) ** 2 for a in v) / len(v)
        return (v - mu) / math.sqrt(var + 1e-5) * W[p + ".w"] + W[p + ".b"]

    def attend(qs, ks, vs, heads):              # softmax(q k^T / sqrt(hd)) v per head
        C = qs[0].shape[0]
        hd = C // heads
        out = []
        for qv in qs:
            o = np.zeros(C)
            for hh in range(heads):
                sl = slice(hh * hd, (hh + 1) * hd)
                sc = [float(qv[sl] @ kv[sl]) / math.sqrt(hd) for kv in ks]
                mx = max(sc)
                e = [math.exp(s - mx) for s in sc]
                z = math.fsum(e)
                for j, vv in enumerate(vs):
                    o[sl] += e[j] / z * vv[sl]
            out.append(o)
        return out

    def resnet(h, p, temb):                     # ResnetBlock2D
        y = silu(groupnorm(h, p + "norm1", 1e-5))
        y = conv(y, p + "conv1")
        for b in range(h.shape[0]):
            y[b] += mv(W[p + "temb.w"], silu(temb[b]), W[p + "temb.b"])
        y = silu(groupnorm(y, p + "norm2", 1e-5))
        y = conv(y, p + "conv2")
        if p + "skip.w" in W:                   # conv_shortcut (1x1) when C_in != C_out
            sk = np.zeros(h.shape[:3] + (y.shape[3],))
            for b in range(h.shape[0]):
                for yy in range(h.shape[1]):
                    for xx in range(h.shape[2]):
                        sk[b, yy, xx] = mv(W[p + "skip.w"], h[b, yy, xx], W[p + "skip.b"])
        else:
            sk = h
        return sk + y

    def transformer(h, p, depth, heads):        # Transformer2DModel (linear projection)
        nb, H, Wd, C = h.shape
        g = groupnorm(h, p + "norm", 1e-6)
        out = np.zeros_like(h)
        for b in range(nb):
            toks = [mv(W[p + "proj_in.w"], g[b, y, xx], W[p + "proj_in.b"])
                    for y in range(H) for xx in range(Wd)]
            ctx = [text[b, j] for j in range(text.shape[1])]
            for k in range(depth):              # BasicTransformerBlock
                q = f"{p}blk{k}."
                n1 = [layernorm(v, q + "ln1") for v in toks]
                a1 = attend([mv(W[q + "attn1.q"], v) for v in n1],
                            [mv(W[q + "attn1.k"], v) for v in n1],
                            [mv(W[q + "attn1.v"], v) for v in n1], heads)
                toks = [v + mv(W[q + "attn1.o"], a, W[q + "attn1.ob"]) for v, a in zip(toks, a1)]
                n2 = [layernorm(v, q + "ln2") for v in toks]
                a2 = attend([mv(W[q + "attn2.q"], v) for v in n2],
                            [mv(W[q + "attn2.k"], c) for c in ctx],
                            [mv(W[q + "attn2.v"], c) for c in ctx], heads)
                toks = [v + mv(W[q + "attn2.o"], a, W[q + "attn2.ob"]) for v, a in zip(toks, a2)]
                new = []
                for v in toks:                  # FeedForward(GEGLU): hidden, gate = chunk(2)
                    pr = mv(W[q + "ff1.w"], layernorm(v, q + "ln3"), W[q + "ff1.b"])
                    hid, gate = pr[:4 * C], pr[4 * C:]
                    gl = np.array([0.5 * a * (1.0 + math.erf(a / math.sqrt(2.0))) for a in gate])
                    new.append(v + mv(W[q + "ff2.w"], hid * gl, W[q + "ff2.b"]))
                toks = new
            for i, v in enumerate(toks):
                y, xx = divmod(i, Wd)
                out[b, y, xx] = h[b, y, xx] + mv(W[p + "proj_out.w"], v, W[p + "proj_out.b"])
        return out

    # time embedding (+ SDXL "text_time" add embedding: concat[pooled, time_ids proj])
    temb = []
    for b in range(B):
        e = mv(W["time.w2"], silu(mv(W["time.w1"], sinusoid(float(t), ch[0]), W["time.b1"])),
               W["time.b2"])
        if cfg.get("add_embed"):
            tid = np.concatenate([sinusoid(float(v), 256) for v in cond["time_ids"][b]])
            a = np.concatenate([np.asarray(cond["pooled"][b], np.float64), tid])
            e = e + mv(W["add.w2"], silu(mv(W["add.w1"], a, W["add.b1"])), W["add.b2"])
        temb.append(e)
    h = conv(np.stack([np.asarray(x, np.float64)] * B), "conv_in")
    res_samples = [h]
    for i in range(nlev):
        heads = ch[i] // cfg["head_dim"]
        for j in range(nres):
            h = resnet(h, f"down{i}.res{j}.", temb)
            if cfg["tdepth"][i]:
                h = transformer(h, f"down{i}.attn{j}.", cfg["tdepth"][i], heads)
            res_samples.append(h)
        if i < nlev - 1:
            h = conv(h, f"down{i}.ds", stride=2)
            res_samples.append(h)
    h = resnet(h, "mid.res0.", temb)
    h = transformer(h, "mid.attn.", cfg["mid_depth"], ch[-1] // cfg["head_dim"])
    h = resnet(h, "mid.res1.", temb)
    for i in range(nlev):
        lev = nlev - 1 - i
        for j in range(nres + 1):
            skip = res_samples.pop()
            h = np.concatenate([h, skip], axis=-1)          # torch.cat([h, res_hidden], dim=1)
            h = resnet(h, f"up{i}.res{j}.", temb)
            if cfg["tdepth"][lev]:
                h = transformer(h, f"up{i}.attn{j}.", cfg["tdepth"][lev], ch[lev] // cfg["head_dim"])
        if i < nlev - 1:                                    # Upsample2D: nearest x2, conv
            nb, H, Wd, C = h.shape
            up = np.zeros((nb, 2 * H, 2 * Wd, C))
            for y in range(2 * H):
                for xx in range(2 * Wd):
                    up[:, y, xx] = h[:, y // 2, xx // 2]
            h = conv(up, f"up{i}.us")
    assert not res_samples
    h = silu(groupnorm(h, "out.norm", 1e-5))
    return conv(h, "out.conv")


def test_unet_forward_bruteforce():
    """oracle/unet.py's whole-image forward (its band generator with every
    exchange answered alone) against the independent per-element evaluation:
    pins the layer composition (ResBlock / Transformer2D order, GEGLU halves,
    GN / LN eps, add-embedding, skip-concat order, up / down sampling)."""
    cfg = _micro_cfg()
    W = gen.weights(cfg, seed=3)
    x = gen.noise(cfg, seed=4).astype(np.float64)
    c = gen.cond(cfg, seed=5)
    got = OU.UNet(cfg, W).forward_full(x, 601, c)
    ref = _brute_unet(cfg, W, x, 601, c)
    assert got.shape == ref.shape == (2, 8, 8, 4)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(ref))
    assert np.max(np.abs(ref[0] - ref[1])) > 1e-3 * np.max(np.abs(ref))   # CFG rows differ
