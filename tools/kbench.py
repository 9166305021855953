"""Kernel micro-bench (CUDA events, warm, inputs > L2): C5-shaped attention and
GEMMs through the kernel-level C ABI.  Prints TFLOP/s per case."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_04719_b200 import stadi as S  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def attn(Nq, Nkv, B, H, hd):
    d = H * hd
    q = torch.randn(Nq * B, d, device="cuda").to(torch.bfloat16)
    kv = torch.randn(Nkv * B * 2, d, device="cuda").to(torch.bfloat16)
    o = torch.empty(Nq * B, d, device="cuda", dtype=torch.bfloat16)
    ms = timeit(lambda: S.k_attention(0, q, kv, o, Nq, Nkv, B, H, hd,
                                     stream=torch.cuda.current_stream()))
    fl = 4.0 * Nq * Nkv * hd * B * H
    print(f"attn Nq={Nq} Nkv={Nkv} B={B} H={H} hd={hd}: {ms:.3f} ms  {fl / ms / 1e9:.0f} TFLOP/s")


def gemm(M, N, K, epi):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.zeros(N, device="cuda")
    kw = dict(bias=bias, B=2)
    if os.environ.get("STADI_SPLITK", "1") != "0":  # the runtime's split-K workspace
        ws = torch.empty(148 * 128 * 256, device="cuda")
        kw.update(ws=ws, ws_elems=ws.numel())
    if epi in (S.EPI_STORE, S.EPI_GELU):
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        kw.update(out=out, ldo=N)
    elif epi in (S.EPI_RES, S.EPI_GATED_RES):
        res = torch.zeros(M, N, device="cuda")
        gate = torch.ones(2, N, device="cuda")
        kw.update(res=res, ldr=N, gate=gate, gate_bstride=N)
    else:
        out = torch.empty(M, N, device="cuda")
        kw.update(out=out, ldo=N)
    ms = timeit(lambda: S.k_gemm(0, A, W, M, N, K, epi, stream=torch.cuda.current_stream(), **kw))
    print(f"gemm M={M} N={N} K={K} epi={epi}: {ms:.3f} ms  {2.0 * M * N * K / ms / 1e9:.0f} TFLOP/s")


def attn_sweep():
    for hd, H in ((64, 18), (72, 16), (80, 16), (40, 16), (16, 16)):
        attn(16384, 16384, 2, H, hd)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "sweep":
    attn_sweep()
elif __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "gemm":
    for M, N, K, e in [(32768, 3456, 1152, S.EPI_STORE), (32768, 1152, 1152, S.EPI_GATED_RES),
                       (32768, 4608, 1152, S.EPI_GELU), (32768, 1152, 4608, S.EPI_GATED_RES),
                       (8192, 8192, 8192, S.EPI_STORE), (2048, 1280, 1280, S.EPI_STORE),
                       (2048, 10240, 1280, S.EPI_STORE), (2048, 1280, 5120, S.EPI_RES),
                       (8192, 640, 640, S.EPI_STORE), (32768, 320, 2880, S.EPI_F32),
                       (128, 1280, 11520, S.EPI_F32), (512, 1280, 11520, S.EPI_F32),
                       (8192, 320, 2880, S.EPI_F32), (256, 1280, 1280, S.EPI_STORE)]:
        gemm(M, N, K, e)
elif __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "unet":
    # SDXL (C4) / SD-1.5 (C3) shapes at N = 1: transformer GEMMs, implicit 3x3 convs, GroupNorm
    for M, N, K, e in [(2048, 3840, 1280, S.EPI_STORE), (2048, 1280, 1280, S.EPI_RES),
                       (2048, 10240, 1280, S.EPI_STORE), (2048, 1280, 5120, S.EPI_RES),
                       (8192, 1920, 640, S.EPI_STORE), (8192, 640, 640, S.EPI_RES),
                       (8192, 5120, 640, S.EPI_STORE), (8192, 640, 2560, S.EPI_RES),
                       (512, 3840, 1280, S.EPI_STORE), (512, 1280, 5120, S.EPI_RES)]:
        gemm(M, N, K, e)
    for h, W, C, N in [(128, 128, 320, 320), (64, 64, 640, 640), (32, 32, 1280, 1280),
                       (64, 64, 320, 320), (32, 32, 640, 640), (16, 16, 1280, 1280)]:
        B = 2
        P = torch.randn((h + 2) * (W + 2) * B, C, device="cuda").to(torch.bfloat16)
        kp = (9 * C + 63) // 64 * 64
        Wt = (torch.randn(N, kp, device="cuda") / kp ** 0.5).to(torch.bfloat16)
        out = torch.empty(h * W * B, N, device="cuda")
        res = torch.zeros(h * W * B, N, device="cuda")
        bias = torch.zeros(N, device="cuda")
        ws = torch.empty(148 * 128 * 256, device="cuda")
        ms = timeit(lambda: S.k_conv3x3_ex(0, P, Wt, h, W, B, C, N, 0, 1, bias=bias, out=out, ldo=N,
                                           res=res, ldr=N, ws=ws, ws_elems=ws.numel(),
                                           stream=torch.cuda.current_stream()))
        fl = 2.0 * h * W * B * N * 9 * C
        print(f"conv3x3 {h}x{W}x{B} C={C} N={N}: {ms * 1e3:.1f} us  {fl / ms / 1e9:.0f} TFLOP/s")
    # stride-2 (mode 1) and upsample (mode 2) convs: implicit vs im2col + GEMM
    for h, W, C, N, mode in [(128, 128, 320, 320, 1), (64, 64, 640, 640, 1), (64, 64, 320, 320, 1),
                             (32, 32, 1280, 1280, 2), (64, 64, 640, 640, 2),
                             (16, 16, 1280, 1280, 2), (32, 32, 640, 640, 2)]:
        B = 2
        ho, wo = (h // 2, W // 2) if mode == 1 else (2 * h, 2 * W)
        P = torch.randn((h + 2) * (W + 2) * B, C, device="cuda").to(torch.bfloat16)
        kp = (9 * C + 63) // 64 * 64
        Wt = (torch.randn(N, kp, device="cuda") / kp ** 0.5).to(torch.bfloat16)
        out = torch.empty(ho * wo * B, N, device="cuda")
        bias = torch.zeros(N, device="cuda")
        ws = torch.empty(148 * 128 * 256, device="cuda")
        fl = 2.0 * ho * wo * B * N * 9 * C
        for imp in (1, 0):
            ms = timeit(lambda: S.k_conv3x3_ex(0, P, Wt, h, W, B, C, N, mode, imp, bias=bias,
                                               out=out, ldo=N, ws=ws, ws_elems=ws.numel(),
                                               stream=torch.cuda.current_stream()))
            print(f"conv3x3 mode={mode} implicit={imp} {h}x{W}x{B} C={C} N={N}: {ms * 1e3:.1f} us"
                  f"  {fl / ms / 1e9:.0f} TFLOP/s")
    for h, W, C in [(128, 128, 320), (64, 64, 640), (32, 32, 1280), (32, 32, 2560), (64, 64, 320),
                    (16, 16, 1280)]:
        B = 2
        x = torch.randn(h * W * B, C, device="cuda")
        g, bt = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
        st = torch.zeros(B * 64, device="cuda", dtype=torch.float64)
        ws = torch.zeros(592 * 2 * B * 32, device="cuda", dtype=torch.float64)
        tk = torch.zeros(32, device="cuda", dtype=torch.int32)
        y = torch.empty((h + 2) * (W + 2) * B, C, device="cuda", dtype=torch.bfloat16)
        ms = timeit(lambda: S.k_groupnorm(0, x, h, W, B, C, g, bt, 1e-5, 1, 1, st, ws, tk, y,
                                          stream=torch.cuda.current_stream()), reps=50)
        by = h * W * B * C * (4 + 4 + 2)
        print(f"groupnorm {h}x{W}x{B} C={C} (partials + apply): {ms * 1e3:.1f} us  "
              f"{by / ms / 1e6:.0f} GB/s")
elif __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "conv":
    # implicit conv vs im2col + GEMM vs the plain GEMM of the same [M, N, 9C] shape;
    # workspace allocated once (split-K allowed), inputs persistent
    imp = int(os.environ.get("CONV_IMPLICIT", "1"))
    for h, W, C, N in [(64, 64, 320, 320), (128, 128, 320, 320), (32, 32, 640, 640),
                       (32, 32, 1280, 1280)]:
        B = 2
        M, K = h * W * B, 9 * C
        P = torch.randn((h + 2) * (W + 2) * B, C, device="cuda").to(torch.bfloat16)
        Wt = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
        out = torch.empty(M, N, device="cuda")
        res = torch.zeros(M, N, device="cuda")
        bias = torch.zeros(N, device="cuda")
        fl = 2.0 * M * N * K
        ws = torch.empty(148 * 128 * 256, device="cuda")
        ms = timeit(lambda: S.k_conv3x3_ex(0, P, Wt, h, W, B, C, N, 0, imp, bias=bias, out=out,
                                           ldo=N, res=res, ldr=N, ws=ws, ws_elems=ws.numel(),
                                           stream=torch.cuda.current_stream()))
        print(f"conv3x3 implicit={imp} {h}x{W}x{B} C={C} N={N}: {ms * 1e3:.1f} us  "
              f"{fl / ms / 1e9:.0f} TFLOP/s")
        gemm(M, N, K, S.EPI_RES)
elif __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "ln":
    M, d = 32768, 1152
    x = torch.randn(M, d, device="cuda")
    y = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
    sh, sc = torch.randn(2, d, device="cuda"), torch.randn(2, d, device="cuda")
    ms = timeit(lambda: S.k_ln_modulate(0, x, y, M, d, 2, sh, sc, d,
                                        stream=torch.cuda.current_stream()))
    print(f"ln_mod M={M} d={d}: {ms * 1e3:.1f} us  {(M * d * 6) / ms / 1e6:.0f} GB/s")
elif __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "xattn":
    attn(16384, 120, 2, 16, 72)
    attn(4096, 120, 2, 16, 72)
    attn(4096, 77, 2, 8, 40)       # SD-1.5 level 0 cross
    attn(4096, 77, 2, 10, 64)      # SDXL level 1 cross
elif __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "small":
    # latency-bound grids (split-K/V candidates): C2 self, SD-1.5 level 1, SDXL level 1 / 2
    attn(256, 256, 2, 16, 72)
    attn(1024, 1024, 2, 8, 80)
    attn(4096, 4096, 2, 10, 64)
    attn(1024, 1024, 2, 20, 64)
    attn(256, 256, 2, 8, 160)
elif __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "attn":
    attn(16384, 16384, 2, 16, 72)
    attn(4096, 4096, 2, 10, 64)
    attn(4096, 4096, 2, 8, 40)
    attn(1024, 1024, 2, 8, 160)
elif __name__ == "__main__":
    attn(16384, 16384, 2, 16, 72)
    attn(8192, 16384, 2, 16, 72)
    attn(4096, 4096, 2, 10, 64)
    attn(4096, 4096, 2, 8, 40)
    for M, N, K, e in [(32768, 3456, 1152, S.EPI_QKV if False else S.EPI_STORE),
                       (32768, 1152, 1152, S.EPI_GATED_RES), (32768, 1152, 1152, S.EPI_RES),
                       (32768, 4608, 1152, S.EPI_GELU), (32768, 1152, 4608, S.EPI_GATED_RES),
                       (8192, 8192, 8192, S.EPI_STORE), (32768, 3456, 1152, S.EPI_F32)]:
        gemm(M, N, K, e)
