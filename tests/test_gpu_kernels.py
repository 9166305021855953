"""Kernel-level parity (GPU): the tcgen05/TMA bf16 kernels and the SIMT fp32
kernels against the oracle's plain fp64 definitions (oracle/dit.py), at
sizes that span several tiles with ragged tails, plus the degenerate cases.

Tolerances (max |x - ref| / max |ref|):
  bf16 kernels: 1e-2 — operands are exact bf16 values, accumulation is fp32;
    the error is the bf16 rounding of the output (2^-9 relative) and, for
    attention, of P (2^-9) — 1e-2 leaves ~5x headroom.
  fp32 SIMT kernels: 1e-5 (fp32 accumulation over K <= 4608).
"""
import numpy as np
import pytest

from oracle import dit as OD

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2509_04719_b200 import stadi
    return stadi


def _bf(x):  # numpy fp32 -> torch bf16 on GPU, and back the exact values
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda().to(torch.bfloat16)
    return t, t.float().cpu().numpy().astype(np.float64)


def _f32(x):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    return t, t.cpu().numpy().astype(np.float64)


def _rel(a, b):
    v = float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))
    print(f"max-abs-rel={v:.3e}")  # collected into the terminal summary (conftest.py)
    return v


GEMM_SHAPES = [(1, 64, 64), (77, 192, 256), (128, 128, 64), (300, 384, 1152), (1000, 256, 128),
               (513, 3456, 1152), (64, 768, 64), (2048, 1152, 4608)]


@pytest.mark.parametrize("dtype", [0, 1], ids=["bf16", "fp32"])
@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_store_f32_gelu(S, dtype, M, N, K):
    rng = np.random.default_rng(M * 7 + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    bias = (rng.standard_normal(N) * 0.1).astype(np.float32)
    mk = _bf if dtype == 0 else _f32
    tA, nA = mk(A)
    tW, nW = mk(W)
    tb = torch.from_numpy(bias).cuda()
    ref = OD.linear(nA, nW, bias.astype(np.float64))
    tol = 1e-2 if dtype == 0 else 1e-5
    # fp32 output
    out = torch.zeros(M, N, device="cuda")
    S.k_gemm(dtype, tA, tW, M, N, K, S.EPI_F32, bias=tb, out=out, ldo=N, B=1)
    torch.cuda.synchronize()
    assert _rel(out.cpu().numpy(), ref) < 1e-5      # fp32 output: fp32 accumulation only
    # T output, GELU
    outT = torch.zeros(M, N, device="cuda", dtype=tA.dtype)
    S.k_gemm(dtype, tA, tW, M, N, K, S.EPI_GELU, bias=tb, out=outT, ldo=N, B=1)
    torch.cuda.synchronize()
    assert _rel(outT.float().cpu().numpy(), OD.gelu_tanh(ref)) < tol


@pytest.mark.parametrize("dtype", [0, 1], ids=["bf16", "fp32"])
def test_gemm_gated_residual_and_qkv(S, dtype):
    rng = np.random.default_rng(5)
    B, ntok, d = 2, 150, 64
    M, K = ntok * B, d
    mk = _bf if dtype == 0 else _f32
    A = rng.standard_normal((M, K)).astype(np.float32)
    # gated residual, gate row per batch
    W = (rng.standard_normal((d, K)) / 8).astype(np.float32)
    tA, nA = mk(A)
    tW, nW = mk(W)
    bias = (rng.standard_normal(d) * 0.1).astype(np.float32)
    gate = rng.standard_normal((B, 7, d)).astype(np.float32)   # batch stride 7*d
    res0 = rng.standard_normal((M, d)).astype(np.float32)
    res = torch.from_numpy(res0.copy()).cuda()
    S.k_gemm(dtype, tA, tW, M, d, K, S.EPI_GATED_RES, bias=torch.from_numpy(bias).cuda(),
             res=res, ldr=d, gate=torch.from_numpy(gate).cuda(), gate_bstride=7 * d, B=B)
    torch.cuda.synchronize()
    lin = OD.linear(nA, nW, bias.astype(np.float64))
    g = gate[np.arange(M) % B, 0, :].astype(np.float64)
    ref = res0 + g * lin
    assert _rel(res.cpu().numpy() - res0, ref - res0) < 1e-5 * (1 if dtype else 1)
    # QKV scatter into two exchange slots at own rows
    Wq = (rng.standard_normal((3 * d, K)) / 8).astype(np.float32)
    tWq, nWq = mk(Wq)
    ntok_full, tok0 = 400, 123
    q = torch.zeros(M, d, device="cuda", dtype=tA.dtype)
    kva = torch.zeros(ntok_full, B, 2, d, device="cuda", dtype=tA.dtype)
    kvb = torch.zeros_like(kva)
    bq = (rng.standard_normal(3 * d) * 0.1).astype(np.float32)
    S.k_gemm(dtype, tA, tWq, M, 3 * d, K, S.EPI_QKV, bias=torch.from_numpy(bq).cuda(), q=q,
             kv_a=kva, kv_b=kvb, kv_row0=tok0 * B, d=d, B=B)
    torch.cuda.synchronize()
    full = OD.linear(nA, nWq, bq.astype(np.float64))
    tol = 1e-2 if dtype == 0 else 1e-5
    assert _rel(q.float().cpu().numpy(), full[:, :d]) < tol
    for kv in (kva, kvb):
        got = kv.float().cpu().numpy()
        own = got[tok0:tok0 + ntok].reshape(M, 2 * d)
        assert _rel(own, full[:, d:]) < tol
        assert np.all(got[:tok0] == 0) and np.all(got[tok0 + ntok:] == 0)


@pytest.mark.parametrize("M,N,K", [(300, 384, 1152), (77, 192, 256)])
def test_gemm_epilogue_vector_and_scalar_paths_agree(S, M, N, K):
    """The 16-byte / 8-byte epilogue (aligned rows) and the 8-byte / 4-byte one
    (rows padded by 2 elements, so not 16-B / 8-B aligned) evaluate the same
    expressions: bit-identical fp32 residual / fp32 output, identical bf16."""
    rng = np.random.default_rng(M + N)
    tA, _ = _bf(rng.standard_normal((M, K)))
    tW, _ = _bf(rng.standard_normal((N, K)) / np.sqrt(K))
    tb = torch.from_numpy((rng.standard_normal(N) * 0.1).astype(np.float32)).cuda()
    gate = torch.from_numpy(rng.standard_normal((2, N)).astype(np.float32)).cuda()
    res0 = rng.standard_normal((M, N + 2)).astype(np.float32)
    outs = {}
    for ld in (N, N + 2):
        f32 = torch.zeros(M, ld, device="cuda")
        S.k_gemm(0, tA, tW, M, N, K, S.EPI_F32, bias=tb, out=f32, ldo=ld, B=1)
        gl = torch.zeros(M, ld, device="cuda", dtype=torch.bfloat16)
        S.k_gemm(0, tA, tW, M, N, K, S.EPI_GELU, bias=tb, out=gl, ldo=ld, B=1)
        res = torch.from_numpy(np.ascontiguousarray(res0[:, :ld])).cuda()
        S.k_gemm(0, tA, tW, M, N, K, S.EPI_GATED_RES, bias=tb, res=res, ldr=ld, gate=gate,
                 gate_bstride=N, B=2)
        # GEGLU: N / 2 outputs per row; row stride N / 2 + 1 (odd) breaks 4-byte alignment
        gg = torch.zeros(M, N // 2 + (ld - N) // 2, device="cuda", dtype=torch.bfloat16)
        S.k_gemm(0, tA, tW, M, N, K, S.EPI_GEGLU, bias=tb, out=gg, ldo=gg.shape[1], B=1)
        torch.cuda.synchronize()
        outs[ld] = [t[:, :n].float().cpu().numpy()
                    for t, n in ((f32, N), (gl, N), (res, N), (gg, N // 2))]
    for a, b in zip(outs[N], outs[N + 2]):
        assert np.array_equal(a, b)


SPLITK_SHAPES = [(128, 1280, 11520), (256, 320, 2880), (300, 640, 1280), (64, 256, 4608),
                 (1000, 192, 2048)]


@pytest.mark.parametrize("M,N,K", SPLITK_SHAPES)
def test_gemm_split_k(S, M, N, K):
    """With a workspace, GEMMs whose tiles fill <= half the SMs split K: every
    epilogue kind against the oracle, and bitwise reproducible (fixed-order reduce)."""
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    bias = (rng.standard_normal(N) * 0.1).astype(np.float32)
    tA, nA = _bf(A)
    tW, nW = _bf(W)
    tb = torch.from_numpy(bias).cuda()
    ws = torch.empty(16 * M * N, device="cuda")
    wk = dict(ws=ws, ws_elems=ws.numel())
    ref = OD.linear(nA, nW, bias.astype(np.float64))
    outs = []
    for _ in range(2):
        out = torch.zeros(M, N, device="cuda")
        S.k_gemm(0, tA, tW, M, N, K, S.EPI_F32, bias=tb, out=out, ldo=N, B=1, **wk)
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy())
    assert _rel(outs[0], ref) < 1e-5
    assert np.array_equal(outs[0], outs[1])
    nosplit = torch.zeros(M, N, device="cuda")
    S.k_gemm(0, tA, tW, M, N, K, S.EPI_F32, bias=tb, out=nosplit, ldo=N, B=1)
    torch.cuda.synchronize()
    # two fp32 summation orders over K <= 11520, each within 1e-5 of the oracle
    assert _rel(outs[0], nosplit.cpu().numpy().astype(np.float64)) < 3e-5
    outT = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    S.k_gemm(0, tA, tW, M, N, K, S.EPI_GELU, bias=tb, out=outT, ldo=N, B=1, **wk)
    torch.cuda.synchronize()
    assert _rel(outT.float().cpu().numpy(), OD.gelu_tanh(ref)) < 1e-2
    B = 2
    gate = rng.standard_normal((B, N)).astype(np.float32)
    res0 = rng.standard_normal((M, N)).astype(np.float32)
    res = torch.from_numpy(res0.copy()).cuda()
    S.k_gemm(0, tA, tW, M, N, K, S.EPI_GATED_RES, bias=tb, res=res, ldr=N,
             gate=torch.from_numpy(gate).cuda(), gate_bstride=N, B=B, **wk)
    torch.cuda.synchronize()
    g = gate[np.arange(M) % B].astype(np.float64)
    assert _rel(res.cpu().numpy() - res0, g * ref) < 1e-5


ATTN_CASES = [  # Nq, Nkv, B, H, hd
    (1, 64, 1, 4, 16), (32, 64, 1, 4, 16), (200, 1000, 2, 3, 64), (128, 256, 2, 2, 72),
    (300, 777, 2, 2, 72), (128, 120, 2, 16, 72), (256, 384, 1, 1, 80), (1000, 2048, 2, 2, 72),
    (300, 1024, 2, 8, 40), (129, 77, 2, 8, 40),    # SD-1.5 level 0 self / cross (hd 40)
    (64, 256, 2, 8, 160), (200, 77, 2, 8, 160),    # SD-1.5 level 2 (hd 160, one Q tile/CTA)
    (500, 1500, 2, 10, 64), (255, 77, 2, 10, 64),  # SDXL level 1 self / cross (hd 64)
    (257, 129, 1, 1, 16), (300, 200, 2, 4, 80),   # the last: two-CTAs-per-SM variant, ragged
    (200, 128, 2, 4, 80), (64, 1, 1, 2, 72),       # single 128-key tile, P over S (<= 128 keys)
]


@pytest.mark.parametrize("dtype", [0, 1], ids=["bf16", "fp32"])
@pytest.mark.parametrize("Nq,Nkv,B,H,hd", ATTN_CASES)
def test_attention(S, dtype, Nq, Nkv, B, H, hd):
    rng = np.random.default_rng(Nq + Nkv + hd)
    d = H * hd
    q = rng.standard_normal((Nq, B, d)).astype(np.float32)
    kv = rng.standard_normal((Nkv, B, 2, d)).astype(np.float32)
    mk = _bf if dtype == 0 else _f32
    tq, nq = mk(q)
    tkv, nkv = mk(kv)
    o = torch.full((Nq * B, d), float("nan"), device="cuda", dtype=tq.dtype)
    S.k_attention(dtype, tq, tkv, o, Nq, Nkv, B, H, hd)
    torch.cuda.synchronize()
    got = o.float().cpu().numpy().reshape(Nq, B, d)
    # oracle layout [B, n, d]
    ref = OD.attention(nq.transpose(1, 0, 2), nkv[:, :, 0].transpose(1, 0, 2),
                       nkv[:, :, 1].transpose(1, 0, 2), H).transpose(1, 0, 2)
    assert np.all(np.isfinite(got))
    assert _rel(got, ref) < (1e-2 if dtype == 0 else 1e-5)


@pytest.mark.parametrize("hd", [72, 64, 40, 160])
def test_attention_growing_max(S, hd):
    """Keys whose logits grow tile after tile (and a late spike): exercises the
    lazy rescaling of O / l in TMEM (running max moves by > 2^8 several times)."""
    rng = np.random.default_rng(hd)
    Nq, Nkv, B, H = 256, 1200, 1, 2
    d = H * hd
    q = rng.standard_normal((Nq, B, d)).astype(np.float32)
    kv = rng.standard_normal((Nkv, B, 2, d)).astype(np.float32) * 0.3
    ramp = np.linspace(0.2, 6.0, Nkv).astype(np.float32)
    kv[:, :, 0] *= ramp[:, None, None]
    kv[1100, :, 0] *= 4.0
    tq, nq = _bf(q)
    tkv, nkv = _bf(kv)
    o = torch.full((Nq * B, d), float("nan"), device="cuda", dtype=torch.bfloat16)
    S.k_attention(0, tq, tkv, o, Nq, Nkv, B, H, hd)
    torch.cuda.synchronize()
    got = o.float().cpu().numpy().reshape(Nq, B, d)
    ref = OD.attention(nq.transpose(1, 0, 2), nkv[:, :, 0].transpose(1, 0, 2),
                       nkv[:, :, 1].transpose(1, 0, 2), H).transpose(1, 0, 2)
    assert np.all(np.isfinite(got))
    assert _rel(got, ref) < 1e-2


def test_attention_full_size_sampled(S):
    """C5 at N = 1, the launch bench.py times: Nq = Nkv = 16384 tokens, B 2,
    16 heads, hd 72.  The oracle evaluates 48 sampled query rows (every head,
    both batch rows) against the full K/V."""
    Nq = Nkv = 16384
    B, H, hd = 2, 16, 72
    d = H * hd
    g = torch.Generator(device="cuda").manual_seed(7)
    tq = torch.randn(Nq * B, d, device="cuda", generator=g).to(torch.bfloat16)
    tkv = torch.randn(Nkv * B * 2, d, device="cuda", generator=g).to(torch.bfloat16)
    o = torch.empty(Nq * B, d, device="cuda", dtype=torch.bfloat16)
    S.k_attention(0, tq, tkv, o, Nq, Nkv, B, H, hd)
    torch.cuda.synchronize()
    rows = np.random.default_rng(1).choice(Nq, 48, replace=False)
    nq = tq.float().cpu().numpy().astype(np.float64).reshape(Nq, B, d)[rows]
    nkv = tkv.float().cpu().numpy().astype(np.float64).reshape(Nkv, B, 2, d)
    got = o.float().cpu().numpy().reshape(Nq, B, d)[rows]
    ref = OD.attention(nq.transpose(1, 0, 2), nkv[:, :, 0].transpose(1, 0, 2),
                       nkv[:, :, 1].transpose(1, 0, 2), H).transpose(1, 0, 2)
    assert _rel(got, ref) < 1e-2


def test_gemm_full_size_sampled(S):
    """C5 QKV GEMM at N = 1: M = 16384 tokens x B 2, N = 3456, K = 1152; sampled rows."""
    M, N, K = 32768, 3456, 1152
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda", generator=g) * 0.1
    out = torch.empty(M, N, device="cuda")
    S.k_gemm(0, A, W, M, N, K, S.EPI_F32, bias=bias, out=out, ldo=N, B=1)
    torch.cuda.synchronize()
    rows = np.random.default_rng(2).choice(M, 64, replace=False)
    nA = A.float().cpu().numpy().astype(np.float64)[rows]
    ref = OD.linear(nA, W.float().cpu().numpy().astype(np.float64),
                    bias.cpu().numpy().astype(np.float64))
    assert _rel(out.cpu().numpy()[rows], ref) < 1e-5 * 50


@pytest.mark.parametrize("dtype", [0, 1], ids=["bf16", "fp32"])
@pytest.mark.parametrize("M,d,B", [(1, 64, 1), (333, 1152, 2), (64, 64, 2)])
def test_ln_modulate(S, dtype, M, d, B):
    rng = np.random.default_rng(M + d)
    x = (rng.standard_normal((M, d)) * 3 + 1).astype(np.float32)
    mod = rng.standard_normal((B, 6, d)).astype(np.float32)
    tx = torch.from_numpy(x).cuda()
    tm = torch.from_numpy(mod).cuda()
    y = torch.zeros(M, d, device="cuda", dtype=torch.bfloat16 if dtype == 0 else torch.float32)
    S.k_ln_modulate(dtype, tx, y, M, d, B, tm[0, 0], tm[0, 1], 6 * d)
    torch.cuda.synchronize()
    b = np.arange(M) % B
    ref = OD.layernorm(x.astype(np.float64)) * (1 + mod[b, 1]) + mod[b, 0]
    assert _rel(y.float().cpu().numpy(), ref) < (1e-2 if dtype == 0 else 1e-5)


def test_bad_shapes_rejected(S):
    A = torch.zeros(128, 100, device="cuda", dtype=torch.bfloat16)
    W = torch.zeros(64, 100, device="cuda", dtype=torch.bfloat16)
    out = torch.zeros(128, 64, device="cuda")
    with pytest.raises(S.StadiError) as e:
        S.k_gemm(0, A, W, 128, 64, 100, S.EPI_F32, out=out, ldo=64, B=1)   # K % 64 != 0
    assert e.value.status == 1
    q = torch.zeros(128, 48, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(S.StadiError):
        S.k_attention(0, q, q, q, 128, 64, 1, 1, 48)                      # hd 48 unsupported


CONV_CASES = [  # h, W, B, C, N, mode, implicit
    (4, 64, 2, 64, 64, 0, 1), (3, 32, 2, 128, 192, 0, 1), (5, 16, 2, 64, 128, 0, 1),
    (2, 128, 2, 320, 320, 0, 1), (7, 8, 2, 64, 64, 0, 1), (1, 64, 1, 64, 256, 0, 1),
    (4, 16, 2, 64, 128, 1, 0), (3, 8, 2, 64, 64, 2, 0), (6, 12, 2, 4, 64, 0, 0),
    # implicit stride 2 (TMA element strides) and upsample (x2-padded input + stride 1)
    (4, 16, 2, 64, 128, 1, 1), (8, 128, 2, 64, 64, 1, 1), (6, 256, 2, 128, 64, 1, 1),
    (2, 64, 1, 64, 64, 1, 1), (3, 8, 2, 64, 64, 2, 1), (2, 64, 2, 128, 64, 2, 1),
    (5, 32, 2, 64, 192, 2, 1),
]


@pytest.mark.parametrize("dtype", [0, 1], ids=["bf16", "fp32"])
@pytest.mark.parametrize("h,W,B,C,N,mode,implicit", CONV_CASES)
def test_conv3x3(S, dtype, h, W, B, C, N, mode, implicit):
    """3x3 conv from the halo-padded token-major buffer vs the oracle's conv
    (oracle/unet.py conv3x3_valid on the same padded, upsampled input)."""
    from oracle import unet as OU
    rng = np.random.default_rng(h * 100 + W + C + mode)
    P = rng.standard_normal((h + 2, W + 2, B, C)).astype(np.float32)
    P[:, 0] = 0
    P[:, -1] = 0
    w = (rng.standard_normal((N, C, 3, 3)) / np.sqrt(9 * C)).astype(np.float32)
    bias = (rng.standard_normal(N) * 0.1).astype(np.float32)
    kp = (9 * C + 63) // 64 * 64
    wt = np.zeros((N, kp), np.float32)
    wt[:, :9 * C] = w.transpose(0, 2, 3, 1).reshape(N, 9 * C)
    mk = _bf if dtype == 0 else _f32
    tP, nP = mk(P)
    tW, nW = mk(wt)
    nw = nW[:, :9 * C].reshape(N, 3, 3, C).transpose(0, 3, 1, 2)
    tb = torch.from_numpy(bias).cuda()
    ho = h // 2 if mode == 1 else (2 * h if mode == 2 else h)
    wo = W // 2 if mode == 1 else (2 * W if mode == 2 else W)
    out = torch.full((ho * wo * B, N), float("nan"), device="cuda")
    S.k_conv3x3(dtype, tP, tW, h, W, B, C, N, mode, implicit if dtype == 0 else 0, tb, out)
    torch.cuda.synchronize()
    x = nP.transpose(2, 0, 1, 3)                       # [B, h+2, W+2, C]
    if mode == 2:   # nearest x2 of the interior, halo rows stay pre-upsample rows
        inner = x[:, 1:-1, 1:-1].repeat(2, axis=1).repeat(2, axis=2)
        top = x[:, :1, 1:-1].repeat(2, axis=2)
        bot = x[:, -1:, 1:-1].repeat(2, axis=2)
        x = OU.pad_cols(np.concatenate([top, inner, bot], axis=1))
    if mode == 1:
        x = x[:, :-1]
    ref = OU.conv3x3_valid(x, nw, bias.astype(np.float64), 2 if mode == 1 else 1)
    got = out.cpu().numpy().reshape(ho, wo, B, N).transpose(2, 0, 1, 3)
    assert np.all(np.isfinite(got))
    assert _rel(got, ref) < (1e-2 if dtype == 0 else 1e-5)


@pytest.mark.parametrize("implicit,mode", [(1, 0), (0, 0), (0, 1), (0, 2), (1, 1), (1, 2)])
def test_conv3x3_time_bias_and_residual(S, implicit, mode):
    """The U-Net ResBlock conv epilogue (EPI_CONV): out = conv + bias + temb[row % B]
    + res, against the oracle's conv3x3_valid plus the two terms; the 16-byte path
    (aligned ldo / ldr) and the unaligned one (rows padded by 2 floats) must agree
    bit for bit."""
    from oracle import unet as OU
    rng = np.random.default_rng(11 + mode + 10 * implicit)
    h, W, B, C, N = 4, 32, 2, 64, 192
    P = rng.standard_normal((h + 2, W + 2, B, C)).astype(np.float32)
    P[:, 0] = 0
    P[:, -1] = 0
    w = (rng.standard_normal((N, C, 3, 3)) / np.sqrt(9 * C)).astype(np.float32)
    bias = (rng.standard_normal(N) * 0.1).astype(np.float32)
    temb = rng.standard_normal((B, N + 4)).astype(np.float32)     # batch stride N + 4
    kp = (9 * C + 63) // 64 * 64
    wt = np.zeros((N, kp), np.float32)
    wt[:, :9 * C] = w.transpose(0, 2, 3, 1).reshape(N, 9 * C)
    tP, nP = _bf(P)
    tW, nW = _bf(wt)
    nw = nW[:, :9 * C].reshape(N, 3, 3, C).transpose(0, 3, 1, 2)
    ho = h // 2 if mode == 1 else (2 * h if mode == 2 else h)
    wo = W // 2 if mode == 1 else (2 * W if mode == 2 else W)
    M = ho * wo * B
    res0 = rng.standard_normal((M, N + 2)).astype(np.float32)
    outs = {}
    for ld in (N, N + 2):
        out = torch.full((M, ld), float("nan"), device="cuda")
        res = torch.from_numpy(np.ascontiguousarray(res0[:, :ld])).cuda()
        S.k_conv3x3_ex(0, tP, tW, h, W, B, C, N, mode, implicit,
                       bias=torch.from_numpy(bias).cuda(), out=out, ldo=ld, res=res, ldr=ld,
                       gate=torch.from_numpy(temb).cuda(), gate_bstride=N + 4)
        torch.cuda.synchronize()
        outs[ld] = out[:, :N].cpu().numpy()
    assert np.array_equal(outs[N], outs[N + 2])
    x = nP.transpose(2, 0, 1, 3)
    if mode == 2:
        inner = x[:, 1:-1, 1:-1].repeat(2, axis=1).repeat(2, axis=2)
        top = x[:, :1, 1:-1].repeat(2, axis=2)
        bot = x[:, -1:, 1:-1].repeat(2, axis=2)
        x = OU.pad_cols(np.concatenate([top, inner, bot], axis=1))
    if mode == 1:
        x = x[:, :-1]
    conv = OU.conv3x3_valid(x, nw, bias.astype(np.float64), 2 if mode == 1 else 1)
    ref = conv.transpose(1, 2, 0, 3).reshape(M, N) \
        + temb[np.arange(M) % B, :N].astype(np.float64) + res0[:, :N].astype(np.float64)
    assert _rel(outs[N], ref) < 1e-5


@pytest.mark.parametrize("max_ctas", [118, 88, 58, 7])
@pytest.mark.parametrize("M,N,K", [(300, 384, 1152), (2048, 1152, 4608), (128, 1280, 11520)])
def test_gemm_on_emulator_grid(S, max_ctas, M, N, K):
    """Under the occupancy emulator (R24) the runtime launches its
    GEMMs on the free SMs only (max_ctas = SMs - held): single-CTA tiles on a
    shrunk persistent grid and that grid's split-K choice.  Every epilogue kind on
    such grids (20 / 40 / 60 % held and an extreme) against the oracle."""
    rng = np.random.default_rng(M + N + K + max_ctas)
    A = rng.standard_normal((M, K)).astype(np.float32)
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    bias = (rng.standard_normal(N) * 0.1).astype(np.float32)
    tA, nA = _bf(A)
    tW, nW = _bf(W)
    tb = torch.from_numpy(bias).cuda()
    ws = torch.empty(16 * M * N, device="cuda")
    wk = dict(ws=ws, ws_elems=ws.numel(), max_ctas=max_ctas)
    ref = OD.linear(nA, nW, bias.astype(np.float64))
    out = torch.zeros(M, N, device="cuda")
    S.k_gemm(0, tA, tW, M, N, K, S.EPI_F32, bias=tb, out=out, ldo=N, B=1, **wk)
    outT = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    S.k_gemm(0, tA, tW, M, N, K, S.EPI_GELU, bias=tb, out=outT, ldo=N, B=1, **wk)
    gate = rng.standard_normal((2, N)).astype(np.float32)
    res0 = rng.standard_normal((M, N)).astype(np.float32)
    res = torch.from_numpy(res0.copy()).cuda()
    S.k_gemm(0, tA, tW, M, N, K, S.EPI_GATED_RES, bias=tb, res=res, ldr=N,
             gate=torch.from_numpy(gate).cuda(), gate_bstride=N, B=2, **wk)
    torch.cuda.synchronize()
    # fp32 accumulation of exact bf16 products: the rounding error grows with K
    # (and with the split-K partial count a 7-CTA grid picks): 1e-5 per 4608 of K
    tol = 1e-5 * max(1.0, K / 4608)
    assert _rel(out.cpu().numpy(), ref) < tol
    assert _rel(outT.float().cpu().numpy(), OD.gelu_tanh(ref)) < 1e-2
    g = gate[np.arange(M) % 2].astype(np.float64)
    assert _rel(res.cpu().numpy() - res0, g * ref) < tol


@pytest.mark.parametrize("switch,hd", [("STADI_ATTN_ALIAS", 72), ("STADI_ATTN_XTILE", 72),
                                       ("STADI_ATTN_DUAL40", 40)])  # "1": the default
def test_attention_alias_variant(S, switch, hd):
    """The P-over-S variant (STADI_ATTN_ALIAS=1, QUAD == 2: two handoffs per key tile)
    against the oracle, in a subprocess (the switches are read once per process), keys
    growing along the sequence so the lazy rescale fires on later tiles; XTILE=1 (the
    default single-tile cross-attention variant) runs the same multi-tile case through
    the unchanged self-attention path."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, torch, sys; sys.path.insert(0, '.');"
            "from paper_2509_04719_b200 import stadi as S; from oracle import dit as OD;"
            f"rng = np.random.default_rng(9); Nq, Nkv, B, H, hd = 300, 777, 2, 2, {hd}; d = H * hd;"
            "q = torch.from_numpy(rng.standard_normal((Nq, B, d)).astype(np.float32)).cuda().bfloat16();"
            "kvn = rng.standard_normal((Nkv, B, 2, d)).astype(np.float32);"
            "kvn[:, :, 0] *= np.linspace(0.5, 40.0, Nkv, dtype=np.float32)[:, None, None];"
            "kv = torch.from_numpy(kvn).cuda().bfloat16();"
            "o = torch.empty(Nq * B, d, device='cuda', dtype=torch.bfloat16);"
            "S.k_attention(0, q, kv, o, Nq, Nkv, B, H, hd); torch.cuda.synchronize();"
            "nq = q.float().cpu().numpy().astype(np.float64); nkv = kv.float().cpu().numpy().astype(np.float64);"
            "ref = OD.attention(nq.transpose(1, 0, 2), nkv[:, :, 0].transpose(1, 0, 2), nkv[:, :, 1].transpose(1, 0, 2), H).transpose(1, 0, 2);"
            "got = o.float().cpu().numpy().reshape(Nq, B, d);"
            "print(float(np.max(np.abs(got - ref)) / np.max(np.abs(ref))))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       env=dict(os.environ, **{switch: "1"}), timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) < 1e-2


GN_SHAPES = [(3, 5, 1, 320), (7, 9, 2, 320), (64, 64, 2, 320), (16, 16, 2, 960),
             (8, 8, 2, 2560), (32, 32, 2, 1920), (1, 1, 2, 64), (33, 17, 2, 640)]


@pytest.mark.parametrize("dtype", [0, 1], ids=["bf16", "fp32"])
@pytest.mark.parametrize("h,W,B,C", GN_SHAPES)
def test_groupnorm(S, dtype, h, W, B, C):
    """GroupNorm partial sums + apply (+SiLU, into the padded conv input) against
    oracle/unet.py gn_partials / gn_apply (R17), inputs with a channel-wise mean
    offset (the variance clamp / cancellation case); bitwise reproducible."""
    from oracle import unet as OU
    rng = np.random.default_rng(h * 1000 + W * 10 + C)
    x = (rng.standard_normal((h, W, B, C)) * 2.0 + rng.standard_normal(C) * 3.0).astype(np.float32)
    gamma = (1.0 + 0.2 * rng.standard_normal(C)).astype(np.float32)
    beta = (0.1 * rng.standard_normal(C)).astype(np.float32)
    xb = np.transpose(x.astype(np.float64), (2, 0, 1, 3))  # oracle layout [B, h, W, C]
    s1, s2, n = OU.gn_partials(xb)
    for act in (0, 1):
        ref = OU.gn_apply(xb, (s1, s2, n), gamma.astype(np.float64), beta.astype(np.float64), 1e-5)
        if act:
            ref = ref / (1.0 + np.exp(-ref))
        ref = np.transpose(ref, (1, 2, 0, 3))  # [h, W, B, C]
        tx = torch.from_numpy(x).cuda()
        tg, tb = torch.from_numpy(gamma).cuda(), torch.from_numpy(beta).cuda()
        stats = torch.zeros(B * 32 * 2, device="cuda", dtype=torch.float64)
        ws = torch.zeros(592 * 2 * B * 32, device="cuda", dtype=torch.float64)
        ticket = torch.zeros(32, device="cuda", dtype=torch.int32)
        odt = torch.bfloat16 if dtype == 0 else torch.float32
        for pad in (0, 1):
            shape = (h + 2, W + 2, B, C) if pad else (h, W, B, C)
            out = torch.full(shape, 7.0, device="cuda", dtype=odt)
            outs = []
            for _ in range(2):
                S.k_groupnorm(dtype, tx, h, W, B, C, tg, tb, 1e-5, act, pad, stats, ws, ticket,
                              out)
                torch.cuda.synchronize()
                outs.append((out.float().cpu().numpy().copy(), stats.cpu().numpy().copy()))
            assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
            st = outs[0][1].reshape(B, 32, 2)
            assert np.allclose(st[..., 0], s1, rtol=1e-5, atol=1e-6 * n[0, 0])
            assert np.allclose(st[..., 1], s2, rtol=1e-5)
            got = outs[0][0]
            if pad:
                assert np.all(got[1:-1, 0] == 0) and np.all(got[1:-1, -1] == 0)
                assert np.all(got[0] == 7.0) and np.all(got[-1] == 7.0)  # halo rows untouched
                got = got[1:-1, 1:-1]
            err = _rel(got.astype(np.float64), ref)
            print(f"groupnorm {h}x{W}x{B}x{C} dtype={dtype} act={act} pad={pad}: {err:.2e}")
            assert err <= (1e-2 if dtype == 0 else 1e-5), err
