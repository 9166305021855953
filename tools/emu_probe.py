"""Kernel throughput under the occupancy emulator (a9): C5-shaped attention and
GEMMs at 0/20/40/60% emulated occupancy (expected slowdown ~ 1 / (1 - rho))."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_2509_04719_b200 import stadi as S  # noqa: E402
from synth import configs, gen  # noqa: E402
import kbench  # noqa: E402

cfg = configs.model("tiny_dit")
ctx = S.Context(S.model_desc("tiny_dit", 0), n_local=1)
W = gen.weights(cfg)
ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
import functools  # noqa: E402
print = functools.partial(print, flush=True)  # noqa: A001
kbench.print = print
_st = torch.cuda.Stream()


def _timeit(fn, reps=10):  # stream-local timing: a device sync would wait for the emulator
    with torch.cuda.stream(_st):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


kbench.timeit = _timeit
which = sys.argv[1] if len(sys.argv) > 1 else "attn"
for pct in (0, 20, 40):
    if pct:
        ctx.emulator_start(pct)
    print(f"--- occupancy {pct}%")
    if which == "attn":
        kbench.attn(16384, 16384, 2, 16, 72)
        kbench.attn(4096, 16384, 2, 16, 72)
    else:
        kbench.gemm(32768, 4608, 1152, S.EPI_GELU)
    if pct:
        ctx.emulator_stop()
ctx.close()
