"""Quality proxy (the "w/ Orig." analogue of Table II,
PAPER.md L294-L308): latent PSNR of STADI and of uniform patch parallelism
against the sequential (single-GPU, fresh) run, on random weights, for the
2-GPU occupancy pairs of Fig. 8 (L292: [0,20], [0,40], [0,60] and [35,45],
[30,50], [25,55]) with v = 1 - rho as the speed proxy.  All ranks run on one
GPU in local mode (exchange by device copies; the protocol is the same as the
NCCL mode's).  Random weights make the absolute PSNR meaningless next to the
paper's; the comparison STADI vs PP vs TA-only / SA-only is what it shows.

    python tools/quality_proxy.py [dit_xl2|sd15] [m_base]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_04719_b200 import stadi as S  # noqa: E402
from synth import configs, gen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "dit_xl2"
mb = int(sys.argv[2]) if len(sys.argv) > 2 else 50
mw = 4
cfg = configs.model(name)
W, x, c = gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)
u = configs.rows_per_unit(cfg)
pt = cfg["latent_h"] // u


def run(speed, flags=0):
    ctx = S.Context(S.model_desc(name, S.DTYPE_BF16), n_local=len(speed))
    try:
        ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
        p = S.plan(speed, mb, mw, pt, u, flags=flags)
        out = np.zeros_like(x)
        ctx.run(p, x, c, out)
        return out.astype(np.float64), p.to_dict()
    finally:
        ctx.close()


def psnr(a, ref):
    rng = ref.max() - ref.min()
    mse = np.mean((a - ref) ** 2)
    return float("inf") if mse == 0 else float(10 * np.log10(rng * rng / mse))


ref, _ = run([1 << 20])
rows = []
for occ in ([0, 20], [0, 40], [0, 60], [35, 45], [30, 50], [25, 55]):
    speed = [int(round((1 << 20) * (100 - o) / 100)) for o in occ]
    r = {"occupancy": occ}
    for tag, flags in (("stadi", 0), ("uniform_pp", S.NO_TA | S.NO_SA), ("sa_only", S.NO_TA),
                       ("ta_only", S.NO_SA)):
        out, p = run(speed, flags)
        r[tag] = {"psnr_db": round(psnr(out, ref), 2), "steps": p["steps"], "units": p["units"]}
    rows.append(r)
    print(json.dumps(r), flush=True)
