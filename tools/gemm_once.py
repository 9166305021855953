"""Launch a few GEMM shapes once each (for ncu launch lists)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_04719_b200 import stadi as S  # noqa: E402

ws = torch.empty(148 * 128 * 256, device="cuda")
for M, N, K in [(128, 1280, 11520), (512, 1280, 11520), (256, 1280, 1280), (2048, 1280, 1280)]:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda")
    for split in (1, 0):
        kw = dict(ws=ws, ws_elems=ws.numel()) if split else {}
        S.k_gemm(0, A, W, M, N, K, S.EPI_F32, out=out, ldo=N, B=2, **kw)
torch.cuda.synchronize()
