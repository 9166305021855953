"""Debug helper: tiny U-Net multi-rank runs vs the oracle, per-band errors."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import stadi as OR  # noqa: E402
from paper_2509_04719_b200 import stadi as S  # noqa: E402
from synth import configs, gen  # noqa: E402

cfg = configs.model("tiny_unet")
W, x, c = gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)
seq = {}
CASES = [([1 << 20, 1 << 19], 10, 2, 1, 0), ([1 << 20, 1 << 19], 4, 2, 1, 0),
         ([3, 2, 1], 6, 2, 1, 3), ([3, 2, 1], 2, 2, 1, 3), ([3, 2, 1], 2, 2, 1, 0),
         ([5, 4, 1], 6, 2, 1, 0), ([5, 4, 1], 2, 2, 1, 0), ([3, 1], 2, 2, 1, 1)]
for speed, mb, mw, dtype, flags in CASES:
    u = configs.rows_per_unit(cfg)
    plan = OR.plan_for(cfg, speed, mb, mw, flags=flags)
    ref = OR.run(cfg, gen.weights_bf16(W) if dtype == 0 else W, x, c, plan)
    ctx = S.Context(S.model_desc("tiny_unet", dtype), n_local=len(speed))
    ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
    p = S.plan(speed, mb, mw, cfg["latent_h"] // u, u, flags=flags)
    out = np.zeros_like(x)
    ctx.run(p, x, c, out)
    ctx.close()
    err = np.abs(out - ref).max(axis=(1, 2)) / np.abs(ref).max()
    print(speed, mb, mw, "flags", flags, "rows", plan["rows"], "steps", plan["steps"],
          "max", err.max())
    print("  per-row err:", " ".join(f"{e:.1e}" for e in err))
