"""Pins for oracle/diffusion.py and oracle/dit.py.

Pinned against closed forms (exact-data DDIM, alpha^2+sigma^2=1, log-series
bound on alpha_bar), textbook special cases (GELU-erf, sin/cos at 0), and
brute-force scalar-loop re-evaluations on tiny inputs (attention, patchify,
unpatchify, a full DiT forward).  No GPU.
"""
import math

import numpy as np
import pytest

from oracle import diffusion, dit, schedule, stadi
from synth import configs, gen


# ----------------------------------------------------------- noise schedule
@pytest.mark.parametrize("kind", ["linear", "scaled_linear"])
def test_alpha_bar_closed_forms(kind):
    ab = diffusion.alpha_bar(kind)
    beta = (np.linspace(1e-4, 0.02, 1000) if kind == "linear"
            else np.linspace(0.00085 ** 0.5, 0.012 ** 0.5, 1000) ** 2)
    assert ab.shape == (1000,)
    assert np.all(np.diff(ab) < 0) and 0 < ab[-1] < ab[0] < 1
    assert abs(ab[0] - (1 - beta[0])) < 1e-15
    # log(1-b) = -b - b^2/2 - R, 0 <= R <= b^3/(3(1-b)): bounds log alpha_bar_999
    approx = -beta.sum() - (beta ** 2).sum() / 2
    assert 0 <= approx - math.log(ab[-1]) <= (beta ** 3 / (3 * (1 - beta))).sum() + 1e-12
    for t in (0, 1, 500, 999, -1):
        a, s, _ = diffusion.alpha_sigma(ab, t)
        assert abs(a * a + s * s - 1) < 1e-15


def test_eq3_exact_on_data_point():
    """If eps_theta returns the true noise of x_t = alpha_t x0 + sigma_t eps, Eq. 3
    lands exactly on alpha_t' x0 + sigma_t' eps (the DDIM ODE solution)."""
    ab = diffusion.alpha_bar("linear")
    rng = np.random.default_rng(0)
    x0, eps = rng.standard_normal((2, 64))
    grid = schedule.fast_grid(10)
    for t, tp in zip(grid, grid[1:] + [schedule.FINAL]):
        a, s, _ = diffusion.alpha_sigma(ab, t)
        a2, s2, _ = diffusion.alpha_sigma(ab, tp)
        got = diffusion.ddim_step(ab, a * x0 + s * eps, eps, t, tp)
        np.testing.assert_allclose(got, a2 * x0 + s2 * eps, rtol=0, atol=1e-12)


def test_eq3_composition_stride2():
    """R12: with a fixed eps, one stride-2 step == two stride-1 steps."""
    ab = diffusion.alpha_bar("scaled_linear")
    rng = np.random.default_rng(1)
    x, e = rng.standard_normal((2, 32))
    g = schedule.fast_grid(50)
    one = diffusion.ddim_step(ab, x, e, g[10], g[12])
    two = diffusion.ddim_step(ab, diffusion.ddim_step(ab, x, e, g[10], g[11]), e, g[11], g[12])
    np.testing.assert_allclose(one, two, atol=1e-13)


def test_cfg_special_cases():
    u, c = np.array([1.0, 2.0]), np.array([3.0, 5.0])
    np.testing.assert_allclose(diffusion.cfg_combine(u, c, 0.0), u)
    np.testing.assert_allclose(diffusion.cfg_combine(u, c, 1.0), c)


# ----------------------------------------------------------- primitives
def test_attention_bruteforce():
    rng = np.random.default_rng(2)
    B, n, N, H, hd = 2, 3, 5, 2, 4
    q = rng.standard_normal((B, n, H * hd))
    k = rng.standard_normal((B, N, H * hd))
    v = rng.standard_normal((B, N, H * hd))
    got = dit.attention(q, k, v, H)
    for b in range(B):
        for h in range(H):
            sl = slice(h * hd, (h + 1) * hd)
            for i in range(n):
                w = [math.exp(sum(q[b, i, sl] * k[b, j, sl]) / math.sqrt(hd)) for j in range(N)]
                z = sum(w)
                ref = sum(w[j] / z * v[b, j, sl] for j in range(N))
                np.testing.assert_allclose(got[b, i, sl], ref, atol=1e-12)


def test_gelu_tanh_vs_erf():
    x = np.linspace(-6, 6, 1001)
    exact = np.array([0.5 * t * (1 + math.erf(t / math.sqrt(2))) for t in x])
    assert np.max(np.abs(dit.gelu_tanh(x) - exact)) < 1e-3
    assert dit.gelu_tanh(np.array([0.0]))[0] == 0.0


def test_layernorm_moments():
    x = np.random.default_rng(3).standard_normal((4, 64)) * 5 + 3
    y = dit.layernorm(x)
    np.testing.assert_allclose(y.mean(-1), 0, atol=1e-12)
    np.testing.assert_allclose(y.var(-1), 1, atol=1e-6)


def test_timestep_and_pos_embed_values():
    f = dit.timestep_freq(0)
    assert np.all(f[:128] == 1) and np.all(f[128:] == 0)
    f = dit.timestep_freq(7)
    assert abs(f[0] - math.cos(7)) < 1e-15 and abs(f[128] - math.sin(7)) < 1e-15
    assert abs(f[127] - math.cos(7 * math.exp(-math.log(1e4) * 127 / 128))) < 1e-15
    d, hp, wp = 16, 3, 5
    pe = dit.pos_embed(d, hp, wp)
    for r in range(hp):
        for c in range(wp):
            row = pe[r * wp + c]
            for k in range(4):
                w = 10000.0 ** (-k / 4)
                assert abs(row[k] - math.sin(c * w)) < 1e-15
                assert abs(row[4 + k] - math.cos(c * w)) < 1e-15
                assert abs(row[8 + k] - math.sin(r * w)) < 1e-15
                assert abs(row[12 + k] - math.cos(r * w)) < 1e-15


# ----------------------------------------------------------- brute-force DiT
def _tiny_cfg(cond="class", guidance=None):
    base = dict(family="dit", cond=cond, hidden=8, heads=2, depth=1, patch=2, c_in=2,
                c_out=3, latent_h=4, latent_w=6, guidance=guidance, schedule="linear")
    if cond == "class":
        base.update(num_classes=3, class_label=1)
    else:
        base.update(text_len=2, text_dim=5)
    base["name"] = "brute"
    return base


def _brute_forward(cfg, W, x, t, cond):
    """Scalar-loop DiT forward written from the architecture description
    (SURVEY O4), independent of oracle/dit.py's vectorised code."""
    W = {k: np.asarray(v, np.float64) for k, v in W.items()}
    d, H, p, C = cfg["hidden"], cfg["heads"], cfg["patch"], cfg["c_in"]
    hd = d // H
    Hl, Wl = cfg["latent_h"], cfg["latent_w"]
    hp, wp = Hl // p, Wl // p
    n = hp * wp
    B = 2 if cfg.get("guidance") else 1

    def lin(vec, w, b):
        return [sum(w[o][i] * vec[i] for i in range(len(vec))) + b[o] for o in range(len(b))]

    def silu(v):
        return [a / (1 + math.exp(-a)) for a in v]

    def gelu(v):
        return [0.5 * a * (1 + math.tanh(math.sqrt(2 / math.pi) * (a + 0.044715 * a ** 3))) for a in v]

    def ln(v):
        mu = sum(v) / len(v)
        var = sum((a - mu) ** 2 for a in v) / len(v)
        return [(a - mu) / math.sqrt(var + 1e-6) for a in v]

    def attn(qs, ks, vs):
        out = []
        for qv in qs:
            o = [0.0] * d
            for h in range(H):
                sc = [sum(qv[h * hd + c] * kv[h * hd + c] for c in range(hd)) / math.sqrt(hd) for kv in ks]
                mx = max(sc)
                e = [math.exp(s - mx) for s in sc]
                z = sum(e)
                for c in range(hd):
                    o[h * hd + c] = sum(e[j] / z * vs[j][h * hd + c] for j in range(len(ks)))
            out.append(o)
        return out

    half = 128
    tf = ([math.cos(t * math.exp(-math.log(1e4) * k / half)) for k in range(half)]
          + [math.sin(t * math.exp(-math.log(1e4) * k / half)) for k in range(half)])
    temb = lin(silu(lin(tf, W["t_embed.w1"], W["t_embed.b1"])), W["t_embed.w2"], W["t_embed.b2"])
    eps = np.zeros((B, Hl, Wl, C))
    for b in range(B):
        if cfg["cond"] == "class":
            cvec = [temb[i] + W["y_embed.table"][cond["labels"][b]][i] for i in range(d)]
            m = lin(silu(cvec), W["blocks.0.ada.w"], W["blocks.0.ada.b"])
            fm = lin(silu(cvec), W["final.ada.w"], W["final.ada.b"])
            y = None
        else:
            t0 = lin(silu(temb), W["t_block.w"], W["t_block.b"])
            m = [W["blocks.0.sst"].reshape(-1)[i] + t0[i] for i in range(6 * d)]
            fm = [W["final.sst"][0][i] + temb[i] for i in range(d)] + \
                 [W["final.sst"][1][i] + temb[i] for i in range(d)]
            y = [lin(gelu(lin(list(cond["text"][b][j]), W["caption.w1"], W["caption.b1"])),
                     W["caption.w2"], W["caption.b2"]) for j in range(cfg["text_len"])]
        sh1, sc1, g1, sh2, sc2, g2 = (m[k * d:(k + 1) * d] for k in range(6))
        hs = []
        for r in range(hp):
            for c in range(wp):
                patch = [x[p * r + dy, p * c + dx, ch] for ch in range(C) for dy in range(p) for dx in range(p)]
                e = lin(patch, W["x_embed.w"], W["x_embed.b"])
                q4 = d // 4
                pe = ([math.sin(c * 1e4 ** (-k / q4)) for k in range(q4)]
                      + [math.cos(c * 1e4 ** (-k / q4)) for k in range(q4)]
                      + [math.sin(r * 1e4 ** (-k / q4)) for k in range(q4)]
                      + [math.cos(r * 1e4 ** (-k / q4)) for k in range(q4)])
                hs.append([e[i] + pe[i] for i in range(d)])
        xm = [[a * (1 + sc1[i]) + sh1[i] for i, a in enumerate(ln(hv))] for hv in hs]
        qkv = [lin(v, W["blocks.0.qkv.w"], W["blocks.0.qkv.b"]) for v in xm]
        a = attn([v[:d] for v in qkv], [v[d:2 * d] for v in qkv], [v[2 * d:] for v in qkv])
        pr = [lin(v, W["blocks.0.proj.w"], W["blocks.0.proj.b"]) for v in a]
        hs = [[hs[j][i] + g1[i] * pr[j][i] for i in range(d)] for j in range(n)]
        if y is not None:
            xq = [lin(v, W["blocks.0.xq.w"], W["blocks.0.xq.b"]) for v in hs]
            kv = [lin(v, W["blocks.0.xkv.w"], W["blocks.0.xkv.b"]) for v in y]
            xa = attn(xq, [v[:d] for v in kv], [v[d:] for v in kv])
            xp = [lin(v, W["blocks.0.xproj.w"], W["blocks.0.xproj.b"]) for v in xa]
            hs = [[hs[j][i] + xp[j][i] for i in range(d)] for j in range(n)]
        xm = [[a * (1 + sc2[i]) + sh2[i] for i, a in enumerate(ln(hv))] for hv in hs]
        mlp = [lin(gelu(lin(v, W["blocks.0.fc1.w"], W["blocks.0.fc1.b"])), W["blocks.0.fc2.w"],
                   W["blocks.0.fc2.b"]) for v in xm]
        hs = [[hs[j][i] + g2[i] * mlp[j][i] for i in range(d)] for j in range(n)]
        for j in range(n):
            r, c = divmod(j, wp)
            v = [a * (1 + fm[d + i]) + fm[i] for i, a in enumerate(ln(hs[j]))]
            o = lin(v, W["final.linear.w"], W["final.linear.b"])
            for dy in range(p):
                for dx in range(p):
                    for ch in range(C):
                        eps[b, p * r + dy, p * c + dx, ch] = o[(dy * p + dx) * cfg["c_out"] + ch]
    return eps


@pytest.mark.parametrize("cond,guidance", [("class", None), ("class", 3.0), ("text", 2.0)])
def test_dit_forward_bruteforce(cond, guidance):
    cfg = _tiny_cfg(cond, guidance)
    W = gen.weights(cfg, seed=5)
    x = gen.noise(cfg, seed=6).astype(np.float64)
    c = gen.cond(cfg, seed=7)
    m = dit.DiT(cfg, W)
    got = m.forward_full(x, 501, c)
    ref = _brute_forward(cfg, W, x, 501, c)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-11)


# ----------------------------------------------------------- protocol reductions
def _c1():
    cfg = configs.model("tiny_dit")
    return cfg, gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)


def test_fresh_patch_forward_equals_unpatched():
    """North star: with staleness disabled (all steps layer-synchronous fresh
    exchange, M_warmup = M_base) the patch-parallel run equals the unpatched one."""
    cfg, W, x, c = _c1()
    seq = stadi.sequential(cfg, W, x, c, 10)
    for speed in ([1, 1], [3, 2, 1], [5, 1, 1, 1]):
        p = stadi.plan_for(cfg, speed, 10, 10, flags=1)     # NO_TA keeps everyone in
        out = stadi.run(cfg, W, x, c, p)
        assert np.max(np.abs(out - seq)) / np.max(np.abs(seq)) < 1e-12
        assert sum(p["rows"]) == cfg["latent_h"]            # patch heights sum to H


def test_single_gpu_run_is_sequential():
    cfg, W, x, c = _c1()
    seq = stadi.sequential(cfg, W, x, c, 10)
    out = stadi.run(cfg, W, x, c, stadi.plan_for(cfg, [1], 10, 2))
    assert np.array_equal(out, seq)


def test_stale_run_is_close_but_not_equal():
    """Stale activations make STADI an approximation (Table II PSNR < inf,
    L297-L306): the C1 run differs from sequential, but only slightly."""
    cfg, W, x, c = _c1()
    seq = stadi.sequential(cfg, W, x, c, 10)
    out, trace = stadi.run(cfg, W, x, c, stadi.plan_for(cfg, [2, 1], 10, 2), return_trace=True)
    rel = np.max(np.abs(out - seq)) / np.max(np.abs(seq))
    assert 1e-6 < rel < 5e-2
    # rank 0 did 10 steps, rank 1 did 6 (Eq. 4)
    assert sum(1 for s in trace if s[1] == 0) == 10 and sum(1 for s in trace if s[1] == 1) == 6


def test_time_invariant_activations_make_staleness_exact():
    """Pin of the stale-exchange protocol (Alg. 1, R9-R14) beyond the
    fresh-exchange reduction: when every activation is independent of x_t and t
    (patch embedding and t-embedding weights zeroed; tokens still differ by their
    positional embedding, so K/V rows differ and must be assembled in the right
    order), a stale read equals a fresh one and eps is constant over the steps.
    Then any plan -- stale rounds, a tier-2 rank's stride-2 steps (Eq. 3 composes
    exactly under a constant eps) -- must reproduce the unpatched sequential run."""
    cfg, W, x, c = _c1()
    W = dict(W)
    for k in ("x_embed.w", "t_embed.w1", "t_embed.w2"):
        W[k] = np.zeros_like(W[k])
    seq = stadi.sequential(cfg, W, x, c, 10)
    assert np.std(seq[:, :, 0] - x[:, :, 0], axis=1).min() > 0   # eps varies over rows
    for speed, flags in (([2, 1], 0), ([3, 2, 1], 1), ([5, 1, 4], 0), ([6, 1, 3], 0)):
        p = stadi.plan_for(cfg, speed, 10, 2, flags=flags)
        out = stadi.run(cfg, W, x, c, p)
        assert np.max(np.abs(out - seq)) <= 1e-12 * np.max(np.abs(seq)), (speed, flags)
    # R32 odd K: the slow GPU's stride is the smallest prime factor of K (3 for
    # M_base 11, 7 for M_base 9); Eq. 3 composes exactly over n intervals under a
    # constant eps, so the stale plan must still equal the sequential run
    for mb, n in ((11, 3), (9, 7)):
        seq_n = stadi.sequential(cfg, W, x, c, mb)
        p = stadi.plan_for(cfg, [2, 1], mb, 2)
        assert p["tier"] == [1, 2] and p["sync_period"] == n
        out = stadi.run(cfg, W, x, c, p)
        assert np.max(np.abs(out - seq_n)) <= 1e-12 * np.max(np.abs(seq_n)), mb
    # the pin is sensitive to the time dependence it removes: restoring the
    # t-embedding makes the same stale plan deviate
    W0 = _c1()[1]
    W2 = dict(W, **{"t_embed.w1": W0["t_embed.w1"], "t_embed.w2": W0["t_embed.w2"]})
    seq2 = stadi.sequential(cfg, W2, x, c, 10)
    out2 = stadi.run(cfg, W2, x, c, stadi.plan_for(cfg, [2, 1], 10, 2))
    assert np.max(np.abs(out2 - seq2)) > 1e-9 * np.max(np.abs(seq2))


def test_temporal_redundancy_trend_thm1_thm2():
    """Theorems 1 and 2 (§IV, Eq. 6-7): the single-step
    difference |x_{t_m} - x_{t_{m+1}}| of a GPU's state is O(1/M) -- for a fast
    GPU (Thm 1) and for a slow GPU whose one step spans n = 2 fast-grid
    intervals (Thm 2, n M_i = M).  On the C1 oracle run (speeds [2, 1]: tier 1 +
    tier 2) the largest step difference of each rank must fall with M_base, M d
    must approach a constant (d halves when M doubles, asymptotically), and the
    slow rank's steps must be ~n = 2 times the fast rank's."""
    cfg, W, x, c = _c1()
    d = {}
    for mb in (10, 20, 50, 100):
        p = stadi.plan_for(cfg, [2, 1], mb, 2)
        assert p["tier"] == [1, 2]
        _, trace = stadi.run(cfg, W, x, c, p, return_trace=True)
        prev = {r: x[p["row_begin"][r]:p["row_begin"][r] + p["rows"][r]].astype(np.float64)
                for r in range(2)}
        dm = [0.0, 0.0]
        for _, r, _, band in trace:
            dm[r] = max(dm[r], float(np.max(np.abs(band - prev[r]))))
            prev[r] = band
        d[mb] = dm
    for r in range(2):
        assert d[10][r] > d[20][r] > d[50][r] > d[100][r], (r, d)
        assert 1.6 < d[50][r] / d[100][r] < 2.2, (r, d)        # O(1/M): M d -> const
    for mb in (50, 100):
        assert 1.6 < d[mb][1] / d[mb][0] < 2.5, d               # Thm 2, n = 2


def test_cfg_split_equals_pair_plan():
    """R33: running each CFG branch on its own GPU (B = 1 conditioning, K/V exchanged
    within the branch, eps bands combined per step inside a pair) reproduces the
    unsplit run of the pair plan -- the batch split changes placement only; with
    stale rounds and a tier-2 pair, class (C1 + CFG) and text (tiny PixArt) models."""
    from oracle import planner as OP
    for cfg in (configs.model("tiny_dit", guidance=3.0), _tiny_cfg("text", 2.0)):
        W = gen.weights(cfg, seed=2)
        x = gen.noise(cfg, seed=3).astype(np.float64)
        c = gen.cond(cfg, seed=4)
        u = configs.rows_per_unit(cfg)
        sp = OP.plan_cfg_split([100, 60, 90, 30, 5], 10, 2, cfg["latent_h"] // u, u)
        assert 2 in sp["tier"] and sp["tier"][4] == 0            # tier-2 pair, odd GPU out
        a = stadi.run_cfg_split(cfg, W, x, c, sp)
        b = stadi.run(cfg, W, x, c, sp["pair_plan"])
        assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b))
