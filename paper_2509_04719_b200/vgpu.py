"""Virtual GPUs: N ranks of one request on ONE device, each a libstadi context
confined to a green-context SM partition (stadi_dist_desc.vgpu_sms), one host
thread per rank, exchanging over the IPC transport (in-process peers).

Thread plumbing only -- every step of the path runs inside libstadi's kernels;
the ctypes calls release the GIL, so the ranks' host threads (and their
partitions) run concurrently.  See green.cuh / DESIGN.md for what is and is not
shared between partitions (HBM, L2 and copy engines are).
"""
from __future__ import annotations

import threading

from . import stadi as S


class VirtualGpus:
    """`n` ranks, `sms` SMs each (multiple of 8), on device `device`."""

    def __init__(self, desc, n, sms, weights, device=0):
        self.n = n
        sess = S.ipc_session_id()
        self.ctx = [None] * n
        errs = []

        def mk(r):
            try:
                c = S.Context(desc, rank=r, world=n, device=device, nccl_id=sess,
                              transport=S.TRANSPORT_IPC, vgpu_sms=sms)
                c.load_weights(weights)
                self.ctx[r] = c
            except Exception as e:  # pragma: no cover - surfaced below
                errs.append(e)
        self._par(mk)
        if errs:
            self.close()
            raise errs[0]

    def _par(self, fn):
        th = [threading.Thread(target=fn, args=(r,)) for r in range(self.n)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    def call(self, method, *args, per_rank=None, **kw):
        """Run ctx.<method>(*args) on every rank concurrently (a COLLECTIVE call);
        per_rank(r) -> extra kwargs.  Returns the per-rank results."""
        out = [None] * self.n
        errs = []

        def go(r):
            try:
                extra = per_rank(r) if per_rank else {}
                out[r] = getattr(self.ctx[r], method)(*args, **kw, **extra)
            except Exception as e:
                errs.append(e)
        self._par(go)
        if errs:
            raise errs[0]
        return out

    def close(self):
        for c in self.ctx:
            if c is not None:
                c.close()
        self.ctx = [None] * self.n
