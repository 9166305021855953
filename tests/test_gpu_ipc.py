"""Multi-process STADI over the IPC transport (GPU): 2-4 processes, one rank each,
all on cuda:0 (the test box has one GPU; the same code maps peers on other GPUs
over NVLink on a multi-GPU node).  Bytes really cross between processes here:

* K/V rows are stored by each rank's QKV GEMM epilogue straight into the other
  processes' exchange slots (CUDA IPC mappings), halo rows go to the two
  neighbour ranks, GroupNorm partial sums to all, and every hand-over is a
  stream memory operation on a flag in the receiver's memory (Alg. 1
  L136-L152, L288);
* stale rounds, a tier-2 rank (stride-2 steps) and an excluded rank are covered;
* three requests per process: the first two replay the per-step CUDA graphs
  (flags restart from zero each request), the third runs eager with kernel
  timing, which also measures the exchange-wait time.

Checks: every rank gathers the same full latent; it equals the local-mode run
(all ranks in one process, device copies) bit for bit; it matches the fp64
oracle within the north-star tolerance (the same cached references as
test_gpu_parity / test_gpu_unet).
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

from oracle import planner as OP
from oracle import stadi as OR
from synth import configs, gen
import refcache

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "helpers", "ipc_worker.py")
TOL = {0: 2e-2, 1: 1e-4}

CASES = [  # id, name, kwargs, speeds, m_base, m_warmup, flags, dtype
    ("c1_tier2", "tiny_dit", {}, [1 << 20, 1 << 19], 10, 2, 0, 0),
    ("c1_tier2_fp32", "tiny_dit", {}, [1 << 20, 1 << 19], 10, 2, 0, 1),
    ("c1_excluded", "tiny_dit", {}, [100, 60, 100, 10], 10, 2, 0, 0),
    ("c1_uniform3", "tiny_dit", {}, [3, 2, 1], 10, 2, OP.NO_TA | OP.NO_SA, 0),
    ("c2_depth2", "dit_xl2", dict(depth=2), [65536, 39322], 50, 4, 0, 0),
    ("unet_tier2", "tiny_unet", {}, [1 << 20, 1 << 19], 10, 2, 0, 0),
    ("unet_3ranks", "tiny_unet", {}, [3, 2, 1], 6, 2, OP.NO_TA | OP.NO_SA, 0),
]


@pytest.fixture(scope="module")
def S():
    from paper_2509_04719_b200 import stadi
    return stadi


def _oracle(cfg, W, x, c, plan, dtype):
    key = dict(kind="stadi_run", cfg=cfg, dtype=dtype, plan=plan)
    return refcache.cached(key, lambda: OR.run(cfg, gen.weights_bf16(W) if dtype == 0 else W,
                                               x, c, plan))


def _local(S, name, cfg, W, x, c, speed, mb, mw, flags, dtype):
    depth = cfg.get("depth", 0) if cfg["family"] == "dit" else 0
    ctx = S.Context(S.model_desc(name, dtype, depth=depth, latent_h=cfg["latent_h"],
                                 latent_w=cfg["latent_w"]), n_local=len(speed))
    try:
        ctx.load_weights([W[n] for n, _, _ in configs.manifest(cfg)])
        u = configs.rows_per_unit(cfg)
        p = S.plan(speed, mb, mw, cfg["latent_h"] // u, u, flags=flags)
        out = np.zeros_like(x)
        ctx.run(p, x, c, out)
        return out
    finally:
        ctx.close()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_ipc_multiprocess(S, case):
    cid, name, kw, speed, mb, mw, flags, dtype = case
    world = len(speed)
    sess = S.ipc_session_id()[:16].hex()
    with tempfile.TemporaryDirectory() as d:
        procs = [subprocess.Popen([sys.executable, WORKER, d, str(r), str(world), sess, name,
                                   str(dtype), ",".join(map(str, speed)), str(mb), str(mw),
                                   str(flags), json.dumps(kw), "3"],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
                 for r in range(world)]
        logs = []
        try:
            for p in procs:
                logs.append(p.communicate(timeout=420)[0])
        finally:
            for p in procs:
                if p.poll() is None:
                    p.kill()
        for r, p in enumerate(procs):
            assert p.returncode == 0, f"rank {r} failed:\n{logs[r][-3000:]}"
        outs = [np.load(os.path.join(d, f"rank{r}.npy")) for r in range(world)]
        meta = [json.load(open(os.path.join(d, f"rank{r}.json"))) for r in range(world)]
    for r in range(world):
        for q in range(3):                       # every rank, every request: same image
            assert np.array_equal(outs[r][q], outs[0][0]), (r, q)
    cfg = configs.model(name, **kw)
    W, x, c = gen.weights(cfg), gen.noise(cfg), gen.cond(cfg)
    loc = _local(S, name, cfg, W, x, c, speed, mb, mw, flags, dtype)
    assert np.array_equal(outs[0][0], loc), "IPC multi-process must equal local mode bit for bit"
    plan = OR.plan_for(cfg, speed, mb, mw, flags=flags)
    assert meta[0]["plan"]["steps"] == plan["steps"] and meta[0]["plan"]["rows"] == plan["rows"]
    ref = _oracle(cfg, W, x, c, plan, dtype)
    err = float(np.max(np.abs(outs[0][0].astype(np.float64) - ref)) / np.max(np.abs(ref)))
    inc = [r for r in range(world) if plan["tier"][r]]
    xb = [m["stats"][-1]["exchange_bytes"] for m in meta]
    wt = [round(m["stats"][-1]["ms_exchange_wait"], 3) for m in meta]
    gs = [m["stats"][1]["graph_steps"] for m in meta]     # second request: graph replays
    print(f"IPC {cid}: {world} processes on one GPU, steps={plan['steps']} rows={plan['rows']} "
          f"max-abs-rel={err:.3e} exchange_bytes={xb} exchange_wait_ms={wt} graph_steps={gs}")
    assert err <= TOL[dtype]
    for r in inc:
        if len(inc) > 1:
            assert xb[r] > 0                     # bytes did cross between processes


def test_ipc_watchdog_lost_peer(S):
    """SURVEY §5 failure detection: a peer that installs the plan and then vanishes
    must not hang the survivor.  Its request's flag waits never complete; the host
    watchdog (STADI_EXCHANGE_TIMEOUT_S) releases the waits, poisons the context and
    stadi_run returns an error; close() then returns."""
    sess = S.ipc_session_id()[:16].hex()
    env = dict(os.environ, STADI_EXCHANGE_TIMEOUT_S="5")
    with tempfile.TemporaryDirectory() as d:
        args = [d, "", "2", sess, "tiny_dit", "0", f"{1 << 20},{1 << 19}", "10", "2", "0", "{}", "1"]
        procs = []
        for r, role in ((0, "survive"), (1, "die")):
            a = list(args)
            a[1] = str(r)
            procs.append(subprocess.Popen([sys.executable, WORKER] + a + [role], env=env,
                                          stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                          text=True))
        try:
            logs = [p.communicate(timeout=180)[0] for p in procs]
        finally:
            for p in procs:
                if p.poll() is None:
                    p.kill()
        assert procs[0].returncode == 0, logs[0][-2000:]
        res = json.load(open(os.path.join(d, "rank0.json")))
    print(f"IPC watchdog: survivor saw {res['watchdog']}")
    assert res["watchdog"].startswith("error")   # an error, not a hang (watchdog or lost peer)
