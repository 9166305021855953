"""Host-side logic of the multi-GPU (NCCL mode) path, on CPU.

One process per GPU issues, at every exchange site of every PUBLISHING step, one
collective on its communicator; fast ranks' odd steps publish nothing (Alg. 1
L142-146, R10).  NCCL needs every rank of the communicator to issue the same
collectives in the same order, so the included ranks' publish sequences
(pub_ver of each schedule entry, in order) must be identical.  Checked here
through the C ABI's stadi_schedule for random plans, and once more across two
real processes with torch.distributed (gloo, world size 2), the bootstrap the
bench uses (rank 0's id broadcast, max-over-ranks timing).
"""
import os
import random

import pytest

from oracle import planner as OP

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def S():
    from paper_2509_04719_b200 import stadi
    return stadi


def _pub_seq(S, p, r):
    return [st[5] for st in S.schedule(p, r) if st[5] >= 0]


def test_publish_sequences_identical_across_ranks(S):
    rng = random.Random(5)
    checked = 0
    for _ in range(400):
        n = rng.randint(1, 8)
        speed = [rng.randint(1, 1000) for _ in range(n)]
        mb = rng.choice([10, 20, 50, 100])
        mw = rng.choice([2, 4])
        flags = rng.choice([0, 0, OP.NO_TA, OP.NO_SA, OP.SIZER_INTERVAL])
        try:
            p = S.plan(speed, mb, mw, 32, 4, flags=flags)
        except S.StadiError:
            continue
        d = p.to_dict()
        inc = [r for r in range(n) if d["tier"][r]]
        seqs = [_pub_seq(S, p, r) for r in inc]
        assert all(s == seqs[0] for s in seqs)
        # versions are published once each, in order, and every read version
        # was published (or is the warmup chain) before it is read
        assert seqs[0] == sorted(seqs[0]) and len(set(seqs[0])) == len(seqs[0])
        assert len(seqs[0]) == d["n_exchange_rounds"]
        for r in inc:
            seen = set()
            for st in S.schedule(p, r):
                if st[5] >= 0:
                    seen.add(st[5])
                assert st[4] in seen or st[4] == st[5]
        checked += 1
    assert checked > 200


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_04719_b200 import stadi as S
    # rank 0's unique-id-like token reaches every rank (bench.py bootstrap)
    obj = [b"id-from-rank-0" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    # the plan is a pure function of speed[] -> identical on every rank
    p = S.plan([1000, 600], 20, 4, 64, 4)
    seq = _pub_seq(S, p, rank)
    allseq = [None] * world
    dist.all_gather_object(allseq, seq)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)   # max-over-ranks timing
    q.put((rank, obj[0], allseq, float(t.item()), p.to_dict()["steps"]))
    dist.destroy_process_group()


def test_two_process_gloo_bootstrap():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(60)
    assert all(p.exitcode == 0 for p in ps)
    for rank, tok, allseq, tmax, steps in res:
        assert tok == b"id-from-rank-0"
        assert allseq[0] == allseq[1] and len(allseq[0]) == 4 + 16 // 2
        assert tmax == 2.0 and steps == [20, 12]
