"""Virtual-GPU smoke run with progress prints (diagnostics for tests/test_gpu_vgpu.py):
C1 on 2 green partitions of 32 SMs, one host thread per rank."""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2509_04719_b200 import stadi as S  # noqa: E402
from synth import configs, gen  # noqa: E402

stage = sys.argv[1] if len(sys.argv) > 1 else "run"
cfg = configs.model("tiny_dit")
W, x, c = gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)
sess = S.ipc_session_id()
n = 2
p = S.plan([1 << 20, 1 << 19], 10, 2, 8, 2)
out = [np.zeros_like(x) for _ in range(n)]
t0 = time.time()


def log(r, m):
    print(f"[{time.time() - t0:6.2f}s] rank {r}: {m}", flush=True)


def work(r):
    try:
        ctx = S.Context(S.model_desc("tiny_dit", 0), rank=r, world=n, device=0, nccl_id=sess,
                        transport=S.TRANSPORT_IPC, vgpu_sms=32)
        log(r, "created")
        ctx.load_weights([W[k] for k, _, _ in configs.manifest(cfg)])
        log(r, "loaded")
        if stage in ("profile", "run", "direct"):
            ms, sp = ctx.profile_warmup(2, n)
            log(r, f"profiled {ms} {sp}")
        if stage == "direct":
            for q in range(2):
                st = ctx.run(p, x, c, out[r])
                log(r, f"direct run {q} done {st.ms_total:.2f} ms")
        if stage == "run":
            ctx.set_plan(p)
            log(r, "plan set")
            ctx.begin(x, c)
            log(r, "begun (enqueued)")
            for i in range(ctx.num_steps()):
                ctx.denoise_step(i)
            log(r, "steps enqueued")
            ctx.gather(out[r])
            log(r, "gather enqueued")
            st = ctx.run(p, x, c, out[r])
            log(r, f"run done {st.ms_total:.2f} ms graph_steps {st.graph_steps}")
        ctx.close()
        log(r, "closed")
    except Exception as e:
        log(r, f"ERROR {e}")


th = [threading.Thread(target=work, args=(r,)) for r in range(n)]
for t in th:
    t.start()
for t in th:
    t.join()
print("equal:", np.array_equal(out[0], out[1]), flush=True)
