"""One rank of a multi-process STADI request over the IPC transport
(tests/test_gpu_ipc.py spawns `world` of these, all on cuda:0).

argv: out_dir rank world session_hex name dtype speeds(csv) m_base m_warmup flags
      [kwargs-json] [requests]
Writes <out_dir>/rank<r>.npy (the gathered full latent of every request,
stacked) and rank<r>.json (run stats).  Imports only the binding and synth/:
the oracle is never touched here.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2509_04719_b200 import stadi as S  # noqa: E402
from synth import configs, gen  # noqa: E402


def main():
    out_dir, rank, world, sess, name, dtype, speeds, mb, mw, flags = sys.argv[1:11]
    kw = json.loads(sys.argv[11]) if len(sys.argv) > 11 else {}
    requests = int(sys.argv[12]) if len(sys.argv) > 12 else 1
    role = sys.argv[13] if len(sys.argv) > 13 else ""   # "die": install the plan, then vanish
    rank, world, dtype, mb, mw, flags = int(rank), int(world), int(dtype), int(mb), int(mw), int(flags)
    speed = [int(v) for v in speeds.split(",")]
    cfg = configs.model(name, **kw)
    W, x, c = gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)
    depth = cfg.get("depth", 0) if cfg["family"] == "dit" else 0
    desc = S.model_desc(name, dtype, depth=depth, latent_h=cfg["latent_h"],
                        latent_w=cfg["latent_w"])
    sid = bytes.fromhex(sess) + bytes(128 - len(sess) // 2)
    ctx = S.Context(desc, rank=rank, world=world, device=0, nccl_id=sid,
                    transport=S.TRANSPORT_IPC)
    try:
        ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
        u = configs.rows_per_unit(cfg)
        ms, sp = ctx.profile_warmup(2, world)          # collective probe through the files
        assert len(ms) == world and all(m > 0 for m in ms)
        p = S.plan(speed, mb, mw, cfg["latent_h"] // u, u, flags=flags)
        if role:
            ctx.set_plan(p)
            if role == "die":
                os._exit(0)                              # a lost peer: no request, no close
            try:                                         # role "survive": the watchdog fires
                ctx.run(p, x, c, np.zeros_like(x))
                status = "completed"
            except S.StadiError as e:
                status = f"error {e.status}: {e}"
            with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
                json.dump(dict(watchdog=status), f)
            return
        outs, stats = [], []
        for q in range(requests):
            ctx.kernel_timing(q == requests - 1)        # last request: eager, timed waits
            out = np.zeros_like(x)
            st = ctx.run(p, x, c, out)
            outs.append(out)
            stats.append(dict(ms_total=st.ms_total, ms_exchange_wait=st.ms_exchange_wait,
                              exchange_bytes=st.exchange_bytes,
                              kernel_launches=st.kernel_launches, steps_run=st.steps_run,
                              graph_steps=st.graph_steps))
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.stack(outs))
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
            json.dump(dict(stats=stats, plan=p.to_dict(), probe_ms=ms), f)
    finally:
        ctx.close()


if __name__ == "__main__":
    main()
