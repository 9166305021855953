"""Thin ctypes binding of libstadi (include/stadi.h, include/stadi_kernels.h).

Argument marshalling only: every step of the hot path runs inside the
library's CUDA kernels.  Names follow the C ABI (``stadi_plan`` ->
``plan``, ...).  Pointers may be numpy arrays (host), torch tensors (host or
device) or raw integers.  There is no fallback: if libstadi.so cannot be
loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libstadi.so")

MAX_GPUS = 64
NO_TA, NO_SA, SIZER_INTERVAL, FORCE_UNITS, SIZER_AFFINE, CFG_SPLIT = 1, 2, 4, 8, 16, 32
STEP_WARMUP, STEP_UNIFORM, STEP_FAST_EVEN, STEP_FAST_ODD, STEP_SLOW = range(5)
T_FINAL = -1
VER_NONE = -1
PRESET = {"tiny_dit": 0, "dit_xl2": 1, "pixart_alpha": 2, "sd15": 3, "sdxl": 4, "tiny_unet": 5}
DTYPE_BF16, DTYPE_FP32_DEBUG = 0, 1
SAMPLER_DDIM, SAMPLER_DDPM, SAMPLER_DPM2M = 0, 1, 2
EPI_STORE, EPI_GELU, EPI_GATED_RES, EPI_RES, EPI_QKV, EPI_F32, EPI_CONV, EPI_GEGLU = range(8)
KCLASS = {"gemm": 0, "attn": 1, "xattn": 2, "norm": 3, "sampler": 4, "xwait": 5}
TRANSPORT_NCCL, TRANSPORT_IPC = 0, 1
STATUS = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ENCCL", 5: "ESTATE",
          6: "EUNSUPPORTED"}


class StadiError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class PlanParams(C.Structure):
    _fields_ = [("n_gpus", C.c_uint32), ("speed", C.POINTER(C.c_uint64)),
                ("m_base", C.c_uint32), ("m_warmup", C.c_uint32),
                ("a_num", C.c_uint32), ("a_den", C.c_uint32),
                ("b_num", C.c_uint32), ("b_den", C.c_uint32),
                ("p_total", C.c_uint32), ("rows_per_unit", C.c_uint32),
                ("flags", C.c_uint32), ("forced_units", C.POINTER(C.c_uint32)),
                ("alpha", C.POINTER(C.c_uint64)), ("beta", C.POINTER(C.c_uint64))]


class Plan(C.Structure):
    _fields_ = [("n_gpus", C.c_uint32), ("m_base", C.c_uint32), ("m_warmup", C.c_uint32),
                ("p_total", C.c_uint32), ("rows_per_unit", C.c_uint32),
                ("tier", C.c_uint8 * MAX_GPUS), ("steps", C.c_uint32 * MAX_GPUS),
                ("units", C.c_uint32 * MAX_GPUS), ("row_begin", C.c_uint32 * MAX_GPUS),
                ("rows", C.c_uint32 * MAX_GPUS), ("sync_period", C.c_uint32),
                ("n_exchange_rounds", C.c_uint32), ("makespan_num", C.c_uint64),
                ("makespan_den", C.c_uint64), ("cfg_split", C.c_uint32),
                ("branch", C.c_uint8 * MAX_GPUS), ("partner", C.c_int8 * MAX_GPUS)]

    def to_dict(self):
        n = self.n_gpus
        return dict(n_gpus=n, m_base=self.m_base, m_warmup=self.m_warmup, p_total=self.p_total,
                    rows_per_unit=self.rows_per_unit, tier=list(self.tier[:n]),
                    steps=list(self.steps[:n]), units=list(self.units[:n]),
                    row_begin=list(self.row_begin[:n]), rows=list(self.rows[:n]),
                    sync_period=self.sync_period, n_exchange_rounds=self.n_exchange_rounds,
                    makespan=(self.makespan_num, self.makespan_den), cfg_split=self.cfg_split,
                    branch=list(self.branch[:n]), partner=list(self.partner[:n]))


class Step(C.Structure):
    _fields_ = [("m", C.c_int32), ("t", C.c_int32), ("t_prev", C.c_int32), ("kind", C.c_int32),
                ("read_ver", C.c_int32), ("pub_ver", C.c_int32)]

    def tuple(self):
        return (self.m, self.t, self.t_prev, self.kind, self.read_ver, self.pub_ver)


class ModelDesc(C.Structure):
    _fields_ = [("preset", C.c_int32), ("dtype", C.c_int32), ("sampler", C.c_int32),
                ("depth", C.c_int32), ("latent_h", C.c_int32), ("latent_w", C.c_int32)]


class DistDesc(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("device", C.c_int32),
                ("n_local", C.c_int32), ("nccl_id", C.POINTER(C.c_uint8)),
                ("transport", C.c_int32), ("vgpu_sms", C.c_int32)]


class Cond(C.Structure):
    _fields_ = [("labels", C.POINTER(C.c_int32)), ("text", C.POINTER(C.c_float)),
                ("pooled", C.POINTER(C.c_float)), ("time_ids", C.POINTER(C.c_float)),
                ("ddpm_seed", C.c_uint64)]


class RunStats(C.Structure):
    _fields_ = [("ms_total", C.c_double), ("ms_exchange_wait", C.c_double),
                ("exchange_bytes", C.c_uint64), ("kernel_launches", C.c_uint32),
                ("steps_run", C.c_uint32), ("graph_steps", C.c_uint32)]


class KEpi(C.Structure):
    _fields_ = [("bias", C.c_void_p), ("out", C.c_void_p), ("ldo", C.c_int32),
                ("res", C.c_void_p), ("ldr", C.c_int32), ("gate", C.c_void_p),
                ("gate_bstride", C.c_int32), ("B", C.c_int32), ("q", C.c_void_p),
                ("kv_a", C.c_void_p), ("kv_b", C.c_void_p), ("kv_row0", C.c_int64),
                ("d", C.c_int32), ("ws", C.c_void_p), ("ws_elems", C.c_int64)]


EXPORTS = [
    "stadi_abi_version", "stadi_status_str", "stadi_last_error", "stadi_plan", "stadi_schedule",
    "stadi_weight_count", "stadi_weight_info", "stadi_create", "stadi_destroy",
    "stadi_load_weights", "stadi_profile_warmup", "stadi_set_plan", "stadi_begin",
    "stadi_num_steps", "stadi_denoise_step", "stadi_gather", "stadi_run",
    "stadi_emulator_start", "stadi_emulator_stop", "stadi_nccl_unique_id",
    "stadi_ipc_session_id", "stadi_profile_band",
    "stadi_kernel_timing", "stadi_kernel_stats",
    "stadi_k_gemm", "stadi_k_gemm_ex", "stadi_k_attention", "stadi_k_ln_modulate",
    "stadi_k_conv3x3", "stadi_k_conv3x3_ex",
    "stadi_k_sampler", "stadi_k_ddpm_noise", "stadi_k_groupnorm", "stadi_k_launch_count",
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2509_04719_b200.build`")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp = C.c_void_p
    sig = {
        "stadi_abi_version": (C.c_uint32, []),
        "stadi_status_str": (C.c_char_p, [C.c_int]),
        "stadi_last_error": (C.c_char_p, [vp]),
        "stadi_plan": (C.c_int, [C.POINTER(PlanParams), C.POINTER(Plan)]),
        "stadi_schedule": (C.c_int, [C.POINTER(Plan), C.c_uint32, C.POINTER(Step), C.c_uint32,
                                     C.POINTER(C.c_uint32)]),
        "stadi_weight_count": (C.c_int, [C.POINTER(ModelDesc), C.POINTER(C.c_uint32)]),
        "stadi_weight_info": (C.c_int, [C.POINTER(ModelDesc), C.c_uint32, C.c_char_p, C.c_uint32,
                                        C.POINTER(C.c_uint64)]),
        "stadi_create": (C.c_int, [C.POINTER(ModelDesc), C.POINTER(DistDesc), C.POINTER(vp)]),
        "stadi_destroy": (None, [vp]),
        "stadi_load_weights": (C.c_int, [vp, C.c_uint32, C.POINTER(vp), C.POINTER(C.c_uint64)]),
        "stadi_profile_warmup": (C.c_int, [vp, C.c_uint32, C.POINTER(C.c_double),
                                           C.POINTER(C.c_uint64)]),
        "stadi_set_plan": (C.c_int, [vp, C.POINTER(Plan)]),
        "stadi_begin": (C.c_int, [vp, vp, C.POINTER(Cond), vp]),
        "stadi_num_steps": (C.c_int, [vp, C.POINTER(C.c_uint32)]),
        "stadi_denoise_step": (C.c_int, [vp, C.c_uint32, vp]),
        "stadi_gather": (C.c_int, [vp, vp, vp]),
        "stadi_run": (C.c_int, [vp, C.POINTER(Plan), vp, C.POINTER(Cond), vp,
                                C.POINTER(RunStats), vp]),
        "stadi_emulator_start": (C.c_int, [vp, C.c_uint32]),
        "stadi_emulator_stop": (C.c_int, [vp]),
        "stadi_nccl_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
        "stadi_ipc_session_id": (C.c_int, [C.POINTER(C.c_uint8)]),
        "stadi_profile_band": (C.c_int, [vp, C.c_uint32, C.POINTER(C.c_uint32),
                                         C.POINTER(C.c_double)]),
        "stadi_kernel_timing": (C.c_int, [vp, C.c_int32]),
        "stadi_kernel_stats": (C.c_int, [vp, C.c_int32, C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]),
        "stadi_k_gemm": (C.c_int, [C.c_int32, vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                   C.POINTER(KEpi), vp]),
        "stadi_k_gemm_ex": (C.c_int, [C.c_int32, vp, vp, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.POINTER(KEpi), C.c_int32, vp]),
        "stadi_k_conv3x3_ex": (C.c_int, [C.c_int32, vp, vp, C.c_int32, C.c_int32, C.c_int32,
                                         C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                         C.POINTER(KEpi), C.c_int32, vp]),
        "stadi_k_attention": (C.c_int, [C.c_int32, vp, vp, vp, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, vp]),
        "stadi_k_ln_modulate": (C.c_int, [C.c_int32, vp, vp, C.c_int32, C.c_int32, C.c_int32, vp,
                                          vp, C.c_int32, vp]),
        "stadi_k_conv3x3": (C.c_int, [C.c_int32, vp, vp, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp]),
        "stadi_k_sampler": (C.c_int, [vp, vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_float,
                                      C.c_float, C.c_float, C.c_uint64, C.c_uint32, C.c_int32,
                                      vp]),
        "stadi_k_ddpm_noise": (C.c_int, [vp, C.c_int64, C.c_uint64, C.c_uint32, C.c_int64, vp]),
        "stadi_k_groupnorm": (C.c_int, [C.c_int32, vp, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, vp, vp, C.c_float, C.c_int32, C.c_int32, vp,
                                        vp, vp, vp, vp]),
        "stadi_k_launch_count": (C.c_uint64, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def _check(st, ctx=None):
    if st != 0:
        msg = lib.stadi_last_error(ctx)
        raise StadiError(st, msg.decode() if msg else "")


def ptr(x):
    """Raw address of a numpy array / torch tensor / int (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    raise TypeError(type(x))


def stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------------- planner
def plan(speed, m_base, m_warmup, p_total, rows_per_unit=1, a=(3, 4), b=(1, 4), flags=0,
         forced_units=None, alpha=None, beta=None) -> Plan:
    n = len(speed)
    sp = (C.c_uint64 * max(n, 1))(*[int(v) for v in speed])
    fu = al = be = None
    if forced_units is not None:
        fu = (C.c_uint32 * n)(*[int(v) for v in forced_units])
    if alpha is not None:
        al = (C.c_uint64 * n)(*[int(v) for v in alpha])
    if beta is not None:
        be = (C.c_uint64 * n)(*[int(v) for v in beta])
    pp = PlanParams(n, C.cast(sp, C.POINTER(C.c_uint64)), m_base, m_warmup, a[0], a[1], b[0],
                    b[1], p_total, rows_per_unit, flags,
                    C.cast(fu, C.POINTER(C.c_uint32)) if fu is not None else None,
                    C.cast(al, C.POINTER(C.c_uint64)) if al is not None else None,
                    C.cast(be, C.POINTER(C.c_uint64)) if be is not None else None)
    out = Plan()
    _check(lib.stadi_plan(C.byref(pp), C.byref(out)))
    return out


def schedule(p: Plan, rank: int):
    n = C.c_uint32(0)
    _check(lib.stadi_schedule(C.byref(p), rank, None, 0, C.byref(n)))
    buf = (Step * max(n.value, 1))()
    _check(lib.stadi_schedule(C.byref(p), rank, buf, n.value, C.byref(n)))
    return [buf[i].tuple() for i in range(n.value)]


def model_desc(preset, dtype=DTYPE_BF16, depth=0, latent_h=0, latent_w=0,
               sampler=SAMPLER_DDIM) -> ModelDesc:
    return ModelDesc(PRESET[preset] if isinstance(preset, str) else preset, dtype, sampler, depth,
                     latent_h, latent_w)


def weight_manifest(desc: ModelDesc):
    n = C.c_uint32(0)
    _check(lib.stadi_weight_count(C.byref(desc), C.byref(n)))
    out = []
    buf = C.create_string_buffer(256)
    for i in range(n.value):
        ne = C.c_uint64(0)
        _check(lib.stadi_weight_info(C.byref(desc), i, buf, 256, C.byref(ne)))
        out.append((buf.value.decode(), ne.value))
    return out


def nccl_unique_id() -> bytes:
    b = (C.c_uint8 * 128)()
    _check(lib.stadi_nccl_unique_id(b))
    return bytes(b)


def ipc_session_id() -> bytes:
    b = (C.c_uint8 * 128)()
    _check(lib.stadi_ipc_session_id(b))
    return bytes(b)


class Context:
    """One stadi_ctx (one process; hosts one rank or n_local ranks on one device)."""

    def __init__(self, desc: ModelDesc, rank=0, world=1, device=0, n_local=1, nccl_id=None,
                 transport=TRANSPORT_NCCL, vgpu_sms=0):
        self._keep = []
        nid = None
        if nccl_id is not None:
            nb = (C.c_uint8 * 128)(*nccl_id)
            self._keep.append(nb)
            nid = C.cast(nb, C.POINTER(C.c_uint8))
        dd = DistDesc(rank, world, device, n_local, nid, transport, vgpu_sms)
        h = C.c_void_p()
        _check(lib.stadi_create(C.byref(desc), C.byref(dd), C.byref(h)))
        self.h = h
        self.desc = desc

    def close(self):
        if getattr(self, "h", None):
            lib.stadi_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def _c(self, st):
        _check(st, self.h)

    def load_weights(self, tensors):
        """tensors: list of float32 C-contiguous numpy arrays in manifest order."""
        arrs = [np.ascontiguousarray(t, dtype=np.float32) for t in tensors]
        ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        ns = (C.c_uint64 * len(arrs))(*[a.size for a in arrs])
        self._c(lib.stadi_load_weights(self.h, len(arrs), ptrs, ns))

    def profile_warmup(self, n_steps, group):
        ms = (C.c_double * group)()
        sp = (C.c_uint64 * group)()
        self._c(lib.stadi_profile_warmup(self.h, n_steps, ms, sp))
        return list(ms), list(sp)

    def profile_band(self, n_steps, units):
        """Compute-only probe step ms of every rank's forced band (units per rank)."""
        u = (C.c_uint32 * len(units))(*[int(v) for v in units])
        ms = (C.c_double * len(units))()
        self._c(lib.stadi_profile_band(self.h, n_steps, u, ms))
        return list(ms)

    def set_plan(self, p: Plan):
        self._c(lib.stadi_set_plan(self.h, C.byref(p)))

    @staticmethod
    def _cond(cond):
        keep = []

        def fptr(x):
            if x is None:
                return None
            if hasattr(x, "data_ptr"):   # torch tensor (host, pinned or device)
                assert x.is_contiguous() and str(x.dtype) == "torch.float32"
                keep.append(x)
                return C.cast(C.c_void_p(x.data_ptr()), C.POINTER(C.c_float))
            a = np.ascontiguousarray(x, dtype=np.float32)
            keep.append(a)
            return a.ctypes.data_as(C.POINTER(C.c_float))

        lp = None
        labels = cond.get("labels")
        if labels is not None:
            la = np.ascontiguousarray(labels, dtype=np.int32)
            keep.append(la)
            lp = la.ctypes.data_as(C.POINTER(C.c_int32))
        tid = cond.get("time_ids")
        if tid is not None and hasattr(tid, "cpu"):
            tid = tid.cpu().numpy()
        return Cond(lp, fptr(cond.get("text")), fptr(cond.get("pooled")), fptr(tid),
                    int(cond.get("ddpm_seed", 0))), keep

    def begin(self, noise, cond, stream=None):
        c, keep = self._cond(cond)
        self._c(lib.stadi_begin(self.h, ptr(noise), C.byref(c), stream_ptr(stream)))

    def num_steps(self):
        n = C.c_uint32(0)
        self._c(lib.stadi_num_steps(self.h, C.byref(n)))
        return n.value

    def denoise_step(self, i, stream=None):
        self._c(lib.stadi_denoise_step(self.h, i, stream_ptr(stream)))

    def gather(self, out, stream=None):
        self._c(lib.stadi_gather(self.h, ptr(out), stream_ptr(stream)))

    def run(self, p: Plan, noise, cond, out, stream=None) -> RunStats:
        c, keep = self._cond(cond)
        st = RunStats()
        self._c(lib.stadi_run(self.h, C.byref(p), ptr(noise), C.byref(c), ptr(out), C.byref(st),
                              stream_ptr(stream)))
        return st

    def emulator_start(self, pct):
        self._c(lib.stadi_emulator_start(self.h, pct))

    def emulator_stop(self):
        self._c(lib.stadi_emulator_stop(self.h))

    def kernel_timing(self, enable=True):
        self._c(lib.stadi_kernel_timing(self.h, 1 if enable else 0))

    def kernel_stats(self, kclass):
        """(launches, ms, algorithmic flops, algorithmic bytes) of a kernel class."""
        n, ms, fl, by = C.c_uint64(), C.c_double(), C.c_double(), C.c_double()
        k = KCLASS[kclass] if isinstance(kclass, str) else kclass
        self._c(lib.stadi_kernel_stats(self.h, k, C.byref(n), C.byref(ms), C.byref(fl),
                                       C.byref(by)))
        return n.value, ms.value, fl.value, by.value


# ---------------------------------------------------------------- kernel-level
def _kepi(ep):
    e = KEpi()
    for k, v in ep.items():
        setattr(e, k, ptr(v) if k in ("bias", "out", "res", "gate", "q", "kv_a", "kv_b", "ws")
                else v)
    return e


def k_gemm(dtype, A, W, M, N, K, epi, stream=None, max_ctas=0, **ep):
    e = _kepi(ep)
    _check(lib.stadi_k_gemm_ex(dtype, ptr(A), ptr(W), M, N, K, epi, C.byref(e), max_ctas,
                               stream_ptr(stream)))


def k_attention(dtype, q, kv, o, Nq, Nkv, B, H, hd, stream=None):
    _check(lib.stadi_k_attention(dtype, ptr(q), ptr(kv), ptr(o), Nq, Nkv, B, H, hd,
                                 stream_ptr(stream)))


def k_ln_modulate(dtype, x, y, M, d, B, shift, scale, bstride, stream=None):
    _check(lib.stadi_k_ln_modulate(dtype, ptr(x), ptr(y), M, d, B, ptr(shift), ptr(scale),
                                   bstride, stream_ptr(stream)))


def k_conv3x3(dtype, P, Wt, h, W, B, C_, N, mode, implicit, bias, out, stream=None):
    _check(lib.stadi_k_conv3x3(dtype, ptr(P), ptr(Wt), h, W, B, C_, N, mode, implicit, ptr(bias),
                               ptr(out), stream_ptr(stream)))


def k_conv3x3_ex(dtype, P, Wt, h, W, B, C_, N, mode, implicit, stream=None, max_ctas=0, **ep):
    """Conv with the full EPI_CONV epilogue: ep = bias, out, ldo, res, ldr, gate,
    gate_bstride (stadi_k_conv3x3_ex)."""
    e = _kepi(ep)
    _check(lib.stadi_k_conv3x3_ex(dtype, ptr(P), ptr(Wt), h, W, B, C_, N, mode, implicit,
                                  C.byref(e), max_ctas, stream_ptr(stream)))


def k_sampler(x, eps_raw, rows, W, C_, p, c_out, ld, B, guidance, A, Bc, Cz=0.0, seed=0, m=0,
              row0=0, stream=None):
    _check(lib.stadi_k_sampler(ptr(x), ptr(eps_raw), rows, W, C_, p, c_out, ld, B, guidance, A,
                               Bc, Cz, seed, m, row0, stream_ptr(stream)))


def k_ddpm_noise(out, n, seed, m, e0=0, stream=None):
    _check(lib.stadi_k_ddpm_noise(ptr(out), n, seed, m, e0, stream_ptr(stream)))


def k_groupnorm(dtype, x, h, W, B, C_, gamma, beta, eps, act, pad, stats, ws, ticket, out,
                stream=None):
    _check(lib.stadi_k_groupnorm(dtype, ptr(x), h, W, B, C_, ptr(gamma), ptr(beta), eps, act, pad,
                                 ptr(stats), ptr(ws), ptr(ticket), ptr(out), stream_ptr(stream)))


def launch_count() -> int:
    return int(lib.stadi_k_launch_count())
