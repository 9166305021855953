"""Launch the C5 attention kernel a few times (for ncu captures)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_04719_b200 import stadi as S  # noqa: E402

Nq = Nkv = 16384
B, H, hd = 2, 16, int(sys.argv[1]) if len(sys.argv) > 1 else 72
H = 1152 // hd if 1152 % hd == 0 else H
d = H * hd
q = torch.randn(Nq * B, d, device="cuda").to(torch.bfloat16)
kv = torch.randn(Nkv * B * 2, d, device="cuda").to(torch.bfloat16)
o = torch.empty(Nq * B, d, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    S.k_attention(0, q, kv, o, Nq, Nkv, B, H, hd)
torch.cuda.synchronize()
