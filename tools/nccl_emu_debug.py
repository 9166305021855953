"""Debug: which call hangs in NCCL mode (single-rank communicator) under the emulator."""
import faulthandler
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["STADI_FORCE_NCCL"] = os.environ.get("STADI_FORCE_NCCL", "1")
from paper_2509_04719_b200 import stadi as S  # noqa: E402
from synth import configs, gen  # noqa: E402

faulthandler.dump_traceback_later(40, exit=True)
t0 = time.time()


def log(*a):
    print(f"[{time.time() - t0:6.1f}s]", *a, flush=True)


cfg = configs.model("tiny_dit")
W, x, c = gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)
ctx = S.Context(S.model_desc("tiny_dit", 0), n_local=1)
log("created")
ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
st = torch.cuda.Stream()
out = np.zeros_like(x)
p = S.plan([1 << 20], 10, 2, 8, 2)
if os.environ.get("PRERUN") == "1":
    ctx.run(p, x, c, out, stream=st)
    log("pre-run")
ctx.profile_warmup(1, 1)
log("probe")
ctx.emulator_start(50)
log("emulator")
ctx.profile_warmup(2, 1)
log("probe under emulator")
ctx.set_plan(p)
log("set_plan")
ctx.begin(x, c, stream=st)
log("begin")
for i in range(ctx.num_steps()):
    ctx.denoise_step(i, stream=st)
    st.synchronize()
    log("step", i)
ctx.gather(out, stream=st)
st.synchronize()
log("gather")
ctx.emulator_stop()
log("stopped")
ctx.close()
