"""Per-kernel-class device time of one request at 0% and 20% emulated occupancy
(which kernels the lost SMs slow down)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_04719_b200 import stadi as S  # noqa: E402
from synth import configs, gen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "sd15"
cfg = configs.model(name)
ctx = S.Context(S.model_desc(name, 0), n_local=1)
W = gen.weights(cfg)
ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
x, c = gen.noise(cfg), gen.cond(cfg)
u = configs.rows_per_unit(cfg)
p = S.plan([1 << 20], 10, 4, cfg["latent_h"] // u, u)
out = np.zeros_like(x)
st = torch.cuda.Stream()
ctx.run(p, x, c, out, stream=st)
ctx.profile_warmup(1, 1)
ctx.run(p, x, c, out, stream=st)
for pct in (0, 20):
    if pct:
        ctx.emulator_start(pct)
    ctx.kernel_timing(True)
    s = ctx.run(p, x, c, out, stream=st)
    st.synchronize()
    ks = {k: ctx.kernel_stats(k) for k in S.KCLASS}
    ctx.kernel_timing(False)
    print(f"{pct}%: request {s.ms_total:.1f} ms", {k: (v[0], round(v[1], 2)) for k, v in ks.items()},
          flush=True)
    if pct:
        ctx.emulator_stop()
ctx.close()
