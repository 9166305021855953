// libstadi runtime: context, weights, plan install, per-request conditioning,
// the patch-parallel DiT step with stale K/V exchange, final gather, run
// loop, speed profiling and the occupancy emulator.
//
// PAPER.md Alg. 1 (L108-L155) is executed as a "program" of steps:
//  * NCCL mode (world > 1, one rank per process): program = this rank's step
//    table (stadi_schedule).  Exchange = grouped ncclBroadcast (one root per
//    rank: an in-place variable-size all-gather, L288) on a side stream.
//  * local mode (world == 1, n_local ranks on one device): program = every
//    hosted rank's steps grouped by fast-grid index m, run layer-lock-step;
//    exchange = device copies of the publisher's rows into the other ranks'
//    slots.  Same kernels, same buffers; used to run the multi-rank protocol
//    (and its parity tests) on one GPU.
//
// Exchange buffers: per attention site l and version
// parity v%2 a full-image K/V slot [N_tok, B, 2, d] (token-major, batch
// innermost, K then V).  A step reading version R publishing P: the QKV GEMM
// epilogue writes the rank's fresh K/V rows into slot[R%2] (so attention sees
// own-fresh + others-stale in one contiguous buffer) and into slot[P%2] (the
// publish), and the exchange delivers the other ranks' rows of version P.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "common.h"
#include "kernels.h"
#include "model.h"

#include <nvtx3/nvToolsExt.h>

namespace {
// NVTX range over one public entry point (SURVEY §5 tracing): the request, its steps,
// the gather and the speed probes show up as named ranges in nsys / ncu timelines;
// a no-op costing a few ns when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  NvtxRange(const char *fmt, unsigned v) {
    char b[64];
    snprintf(b, sizeof b, fmt, v);
    nvtxRangePushA(b);
  }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using namespace stadi;

namespace {

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclCommSplit) CommSplit = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
  decltype(&ncclCommAbort) CommAbort = nullptr;
};
NcclApi &nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
#define LD(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
      LD(GetUniqueId); LD(CommInitRank); LD(CommDestroy); LD(CommSplit); LD(Broadcast);
      LD(AllGather); LD(GroupStart); LD(GroupEnd); LD(GetErrorString); LD(CommGetAsyncError);
      LD(CommAbort);
#undef LD
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast &&
               api.AllGather && api.GroupStart && api.GroupEnd;
    }
  }
  return api;
}

inline int64_t rup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// One hosted rank: its band, activations and exchange slots.
struct Rank {
  int g = 0;                       // group rank (0..G-1)
  int row_begin = 0, rows = 0;     // latent rows
  int tok_begin = 0, n_tok = 0;    // tokens (token rows * wp)
  int tier = 0;
  int branch = 0, partner = -1;    // R33 CFG split: CFG branch and pair partner (group rank)
  std::vector<stadi_step_t> sched;
  float *x_band = nullptr;         // [rows, W, C_in] fp32
  float *hist = nullptr;           // [rows, W, C_in] fp32 previous combined eps (DPM2M, R34)
  float *x_res = nullptr;          // [n_tok*B, d] fp32 residual stream
  void *xmod = nullptr, *q = nullptr, *o = nullptr, *h1 = nullptr;  // T activations
  float *eps_raw = nullptr;        // [n_tok*B, fin_ld] fp32
  std::vector<void *> kv;          // [depth*2] full-image slots
};

struct Part {  // one (hosted rank, schedule entry) executed in a program step
  int li;      // index into ctx->ranks
  stadi_step_t st;
  int idx = 0; // index of the entry in the rank's step table
};

struct UNetState;  // unet_exec.cuh
struct IpcState;   // ipc.cuh

}  // namespace

struct stadi_ctx {
  Dims dm;
  int dtype = STADI_DTYPE_BF16;
  int sampler = STADI_SAMPLER_DDIM;
  uint64_t ddpm_seed = 0;    // per request (stadi_cond), R19
  uint64_t *seed_dev = nullptr;  // device copy of ddpm_seed, read by the sampler kernel so a
                                 // captured step graph serves every request's seed
  int device = 0, rank = 0, world = 1, n_local = 1, G = 1;
  // NCCL mode: one rank per process, exchange by NCCL (world > 1; or world == 1 with
  // STADI_FORCE_NCCL=1, a single-rank communicator that runs the NCCL code path --
  // broadcasts, comm stream, version events, gather -- on one GPU for tests)
  bool nccl = false;
  // IPC mode: one rank per process (world > 1, STADI_TRANSPORT_IPC), one-sided
  // exchange through CUDA IPC mappings of the peers' slots (ipc.cuh)
  bool ipc_mode = false;
  std::unique_ptr<IpcState> ipc;
  bool probe = false;        // profiling probe steps: no exchange waits / signals
  // R33 CFG batch split (plan.cfg_split): every hosted rank runs ONE CFG branch with a
  // forward batch Bf = 1; otherwise Bf = dm.B
  int Bf = 1;
  std::vector<void *> kv_text_b[2];  // per branch: cross-attention text K/V [L, 1, 2, d]
  int ipc_idx = 0;           // IPC mode: step-table index of the step being built / run
  bool kernels_warm = false; // IPC: every kernel of the path loaded (first begin of a ctx)
  uint32_t graph_steps = 0;  // steps replayed from CUDA graphs (stats of stadi_run)
  int num_sms = 148;
  std::string err;
  bool poisoned = false;
  size_t esz = 2;  // element size of T

  // weights
  bool weights_loaded = false;
  std::vector<TensorSpec> man;
  std::vector<void *> wT;    // compute-dtype copy of GEMM weights (nullptr otherwise)
  std::vector<float *> wf;   // fp32 copy (bf16-rounded values in bf16 mode)
  void *ada_all = nullptr;   // [depth*6d, d] T (class presets)
  float *ada_all_b = nullptr;
  float *sst_all = nullptr;  // [depth, 6, d] (text presets)
  void *final_w = nullptr;   // [fin_ld, d] T, zero-padded rows
  float *final_b = nullptr;  // [fin_ld]
  int fin_ld = 64;
  float *pos_full = nullptr; // [hp*wp, d]
  float *splitk_ws = nullptr;  // split-K partial tiles of the small tcgen05 GEMMs
  long splitk_elems = 0;
  std::vector<void *> allocs;

  // plan
  bool has_plan = false;
  stadi_plan_t plan{};
  std::vector<Rank> ranks;   // hosted ranks (included ones)
  std::vector<std::vector<Part>> program;

  // request state
  bool begun = false;
  int n_t = 0;               // = M_base: modulation precomputed for every fast-grid t
  float *mod = nullptr;      // [n_t, B, depth, 6, d]
  float *fmod = nullptr;     // [n_t, B, 2, d]
  float *temb = nullptr, *tmp_f = nullptr, *tfreq = nullptr;
  void *csilu = nullptr;
  int *labels_dev = nullptr;
  size_t cond_cap_nt = 0;
  int tfreq_nt = 0;
  void *text_T = nullptr, *y1 = nullptr, *y = nullptr;
  float *text_f = nullptr;
  std::vector<void *> kv_text;
  double abar[1000];

  // virtual GPU (green-context SM partition, green.cuh): every kernel goes to wstream
  CUgreenCtx green_ctx = nullptr;
  cudaStream_t wstream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  // pinned staging of a request's host <-> device copies (stage_h2d / stage_d2h): no
  // copy from pageable memory, whose implicit synchronisation could wait for another
  // rank's stream (virtual GPUs of one process) or stall the host thread
  char *stage = nullptr;
  size_t stage_cap = 0, stage_off = 0;
  cudaEvent_t stage_ev = nullptr;
  bool stage_pending = false;

  // streams / NCCL
  cudaStream_t comm = nullptr;
  cudaStream_t astream = nullptr;      // stream-ordered plan / request allocations
  cudaStream_t last_stream = nullptr;  // last stream denoise_step / run enqueued on
  bool last_stream_set = false;
  ncclComm_t world_comm = nullptr, sub_comm = nullptr;
  std::vector<cudaEvent_t> ev_done;  // [depth*2] exchange completion per (site, parity)
  std::vector<char> ev_used;
  cudaEvent_t ev_ready = nullptr;
  uint64_t exch_bytes = 0;

  // emulator
  int *emu_flag_dev = nullptr;       // emulator stop flag in DEVICE memory (polling
                                     // host-mapped memory slowed every kernel 3-9x)
  cudaStream_t emu_ctl = nullptr;    // non-blocking stream that writes the flag
  cudaStream_t emu_stream = nullptr;
  int emu_ctas = 0;

  // per-class kernel timing (stadi_kernel_timing): CUDA events recorded on the
  // launching stream around every launch of the class
  struct KClass {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    size_t used = 0;
    uint64_t launches = 0;
    double ms = 0, flops = 0, bytes = 0;
  };
  // CUDA graphs: one per program step of the installed plan (local mode), captured on
  // first use on gstream and replayed on the caller's stream.  Dropped with the plan.
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    unsigned long long launches = 0;  // kernels inside (for the launch counter)
    uint64_t exch_bytes = 0;          // exchange bytes the step moves (counted per replay)
    int emu_ctas = 0;                 // emulator SMs at capture (grid sizes depend on it)
  };
  std::vector<StepGraph> graphs;
  cudaStream_t gstream = nullptr;
  bool ktime = false;
  KClass kt[STADI_KCLASS_COUNT];

  // U-Net family executor state (weights, programs, exchange sites)
  std::unique_ptr<UNetState> un;
};

namespace {

// STADI_DEBUG=1: progress trace of the request calls on stderr (hang diagnostics)
bool debug_on() {
  static const bool v = getenv("STADI_DEBUG") != nullptr;
  return v;
}
#define DBG(...)                                                                         \
  do {                                                                                   \
    if (debug_on()) {                                                                    \
      fprintf(stderr, "[stadi r%d] ", ctx->rank);                                        \
      fprintf(stderr, __VA_ARGS__);                                                      \
      fprintf(stderr, "\n");                                                             \
    }                                                                                    \
  } while (0)

stadi_status ctx_fail(stadi_ctx *c, stadi_status st, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) {
    c->err = buf;
    if (st == STADI_ECUDA || st == STADI_ENCCL) c->poisoned = true;
  }
  tls_error() = buf;
  return st;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return ctx_fail(ctx, STADI_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,     \
                      cudaGetErrorString(e_));                                         \
  } while (0)
#define CKN(call)                                                                      \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess)                                                             \
      return ctx_fail(ctx, STADI_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call,     \
                      nccl().GetErrorString ? nccl().GetErrorString(r_) : "nccl");     \
  } while (0)
#define ALIVE()                                                                        \
  do {                                                                                 \
    if (!ctx) return ctx_fail(nullptr, STADI_EINVAL, "NULL context");                  \
    if (ctx->poisoned) return ctx_fail(ctx, STADI_ESTATE, "context poisoned: %s",      \
                                       ctx->err.c_str());                              \
  } while (0)

#define ST(call)                          \
  do {                                    \
    stadi_status s_ = (call);             \
    if (s_ != STADI_OK) return s_;        \
  } while (0)

// Plan- and request-lifetime device memory is stream-ordered (cudaMallocAsync /
// cudaFreeAsync on the context's allocation stream): re-planning never implies a
// device-wide synchronisation.  That matters because the occupancy emulator
// (a9) keeps a persistent kernel resident — cudaFree / cudaDeviceSynchronize
// would wait for it forever.
template <typename P>
cudaError_t pmalloc(stadi_ctx *ctx, P **p, size_t bytes) {
  void *q = nullptr;
  cudaError_t e = cudaMallocAsync(&q, bytes ? bytes : 16, ctx->astream);
  *p = reinterpret_cast<P *>(q);
  return e;
}
inline void pfree(stadi_ctx *ctx, void *p) {
  if (p) cudaFreeAsync(p, ctx->astream);
}
// Wait for everything this context enqueued (its streams and the caller's last
// stream) without a device-wide synchronisation.
cudaError_t quiesce(stadi_ctx *ctx) {
  cudaError_t e = cudaSuccess;
  if (ctx->last_stream_set) e = cudaStreamSynchronize(ctx->last_stream);
  if (e == cudaSuccess && ctx->comm) e = cudaStreamSynchronize(ctx->comm);
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  if (e == cudaSuccess && ctx->astream) e = cudaStreamSynchronize(ctx->astream);
  if (e == cudaSuccess && ctx->wstream) e = cudaStreamSynchronize(ctx->wstream);
  return e;
}

void ipc_unblock(stadi_ctx *ctx);  // ipc.cuh

// Host wait for an event with a watchdog (SURVEY §5 failure detection): in NCCL mode
// poll ncclCommGetAsyncError; with any exchange transport give up after
// STADI_EXCHANGE_TIMEOUT_S seconds (default 600) -- a dead peer or a broken
// collective then poisons the context (NCCL: the communicators are aborted) instead
// of hanging the process forever.
double exchange_timeout_s() {
  static const double v = [] {
    const char *e = getenv("STADI_EXCHANGE_TIMEOUT_S");
    return e ? atof(e) : 600.0;
  }();
  return v;
}
stadi_status wait_event_watchdog(stadi_ctx *ctx, cudaEvent_t ev) {
  if (!ctx->nccl && !ctx->ipc_mode) {
    const cudaError_t e = cudaEventSynchronize(ev);
    return e == cudaSuccess ? STADI_OK
                            : ctx_fail(ctx, STADI_ECUDA, "event sync: %s", cudaGetErrorString(e));
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t it = 0;; ++it) {
    const cudaError_t e = cudaEventQuery(ev);
    if (e == cudaSuccess) return STADI_OK;
    if (e != cudaErrorNotReady)
      return ctx_fail(ctx, STADI_ECUDA, "event query: %s", cudaGetErrorString(e));
    if (ctx->nccl && nccl().CommGetAsyncError) {
      for (ncclComm_t c : {ctx->world_comm, ctx->sub_comm}) {
        ncclResult_t ar = ncclSuccess;
        if (c && nccl().CommGetAsyncError(c, &ar) == ncclSuccess && ar != ncclSuccess &&
            ar != ncclInProgress) {
          if (nccl().CommAbort) {
            if (ctx->sub_comm && ctx->sub_comm != ctx->world_comm) nccl().CommAbort(ctx->sub_comm);
            if (ctx->world_comm) nccl().CommAbort(ctx->world_comm);
            ctx->sub_comm = ctx->world_comm = nullptr;
          }
          return ctx_fail(ctx, STADI_ENCCL, "NCCL asynchronous error: %s",
                          nccl().GetErrorString ? nccl().GetErrorString(ar) : "?");
        }
      }
    }
    const double el =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > exchange_timeout_s()) {
      if (ctx->nccl && nccl().CommAbort) {
        if (ctx->sub_comm && ctx->sub_comm != ctx->world_comm) nccl().CommAbort(ctx->sub_comm);
        if (ctx->world_comm) nccl().CommAbort(ctx->world_comm);
        ctx->sub_comm = ctx->world_comm = nullptr;
      }
      if (ctx->ipc_mode) ipc_unblock(ctx);  // release this rank's flag waits (results void)
      return ctx_fail(ctx, ctx->nccl ? STADI_ENCCL : STADI_ECUDA,
                      "exchange watchdog: request not complete after %.0f s (peer lost?)", el);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(it < 1000 ? 20 : 200));
  }
}

template <typename P>
cudaError_t dalloc(stadi_ctx *ctx, P **p, size_t bytes) {
  void *q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
  if (e != cudaSuccess) return e;
  ctx->allocs.push_back(q);
  *p = reinterpret_cast<P *>(q);
  return cudaSuccess;
}

bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
bool is_pageable(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// ---------------------------------------------------------------- host staging
// A request's staged copies go through one pinned buffer (sized at create); begin
// waits for the previous request's staged copies, then reuses it from the start.
cudaError_t stage_reset(stadi_ctx *ctx) {
  if (ctx->stage_pending) {
    cudaError_t e = cudaEventSynchronize(ctx->stage_ev);
    if (e != cudaSuccess) return e;
  }
  ctx->stage_pending = false;
  ctx->stage_off = 0;
  return cudaSuccess;
}
char *stage_take(stadi_ctx *ctx, size_t bytes) {
  const size_t off = (ctx->stage_off + 255) / 256 * 256;
  if (off + bytes > ctx->stage_cap) return nullptr;
  ctx->stage_off = off + bytes;
  return ctx->stage + off;
}
// Source pointer for an async host->device copy of `bytes` at src: src itself when it
// is device or pinned memory, else a pinned copy (nullptr: staging exhausted).
const void *stage_h2d(stadi_ctx *ctx, const void *src, size_t bytes) {
  if (!is_pageable(src)) return src;
  char *p = stage_take(ctx, bytes);
  if (p) std::memcpy(p, src, bytes);
  return p;
}
struct D2HCopy {
  void *dst;
  const void *src;
  size_t bytes;
};
void CUDART_CB d2h_finish(void *arg) {  // stream-ordered host copy out of the staging
  D2HCopy *c = static_cast<D2HCopy *>(arg);
  std::memcpy(c->dst, c->src, c->bytes);
  delete c;
}
// Stream-ordered device->host copy into dst (pinned or pageable).
cudaError_t stage_d2h(stadi_ctx *ctx, void *dst, const void *src_dev, size_t bytes,
                      cudaStream_t s) {
  if (!is_pageable(dst))
    return cudaMemcpyAsync(dst, src_dev, bytes, cudaMemcpyDeviceToHost, s);
  char *p = stage_take(ctx, bytes);
  if (!p) return cudaErrorMemoryAllocation;
  cudaError_t e = cudaMemcpyAsync(p, src_dev, bytes, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaLaunchHostFunc(s, d2h_finish, new D2HCopy{dst, p, bytes});
  if (e == cudaSuccess) e = cudaEventRecord(ctx->stage_ev, s);
  ctx->stage_pending = true;
  return e;
}

// ---------------------------------------------------------------- host math (fp64)
void alpha_bar(bool linear, double *ab) {
  double acc = 1.0;
  for (int t = 0; t < 1000; ++t) {
    double beta;
    if (linear) {
      beta = 1e-4 + (0.02 - 1e-4) * t / 999.0;
    } else {
      const double a = std::sqrt(0.00085), b = std::sqrt(0.012);
      const double s = a + (b - a) * t / 999.0;
      beta = s * s;
    }
    acc *= 1.0 - beta;
    ab[t] = acc;
  }
}
// Eq. 3 as x' = A x + Bc eps: A = alpha'/alpha, Bc = -sigma'(e^h - 1).
void ddim_coeffs(const double *ab, int t, int t_prev, float *A, float *Bc) {
  const double a1 = ab[t], a2 = t_prev < 0 ? ab[0] : ab[t_prev];
  const double al = std::sqrt(a1), si = std::sqrt(1 - a1), al2 = std::sqrt(a2),
               si2 = std::sqrt(1 - a2);
  const double h = std::log(al2 / si2) - std::log(al / si);
  *A = (float)(al2 / al);
  *Bc = (float)(-si2 * std::expm1(h));
}

// R19 DDPM (eta = 1) as x' = A x + Bc eps + Cz z:  with x0 = (x - sigma eps) / alpha,
// x' = alpha' x0 + sqrt(1 - abar' - s^2) eps + s z, s = sqrt((1-abar')/(1-abar)) sqrt(1 - abar/abar').
void sampler_coeffs(const stadi_ctx *ctx, int t, int t_prev, float *A, float *Bc, float *Cz) {
  if (ctx->sampler != STADI_SAMPLER_DDPM) {  // DDIM and DPM2M: Eq. 3's A, Bc
    ddim_coeffs(ctx->abar, t, t_prev, A, Bc);
    *Cz = 0.f;
    return;
  }
  const double a1 = ctx->abar[t], a2 = t_prev < 0 ? ctx->abar[0] : ctx->abar[t_prev];
  const double se = std::sqrt((1 - a2) / (1 - a1)) * std::sqrt(1 - a1 / a2);
  *A = (float)(std::sqrt(a2) / std::sqrt(a1));
  *Bc = (float)(std::sqrt(1 - a2 - se * se) - std::sqrt(a2) * std::sqrt(1 - a1) / std::sqrt(a1));
  *Cz = (float)se;
}

// R34 multistep DPM-Solver-2: D = c1 eps + c2 eps_prev, c1 = 1 + 1/(2r), c2 = -1/(2r),
// r = h_prev / h from the band's own previous step (schedule entry idx - 1); the first
// step (idx 0) is Eq. 3 (c2 = 0).
void dpm2m_coeffs(const stadi_ctx *ctx, const std::vector<stadi_step_t> &sched, int idx,
                  float *c1, float *c2) {
  *c1 = 1.f;
  *c2 = 0.f;
  if (ctx->sampler != STADI_SAMPLER_DPM2M || idx <= 0) return;
  auto lam = [&](int t) {
    const double ab = t < 0 ? ctx->abar[0] : ctx->abar[t];
    return 0.5 * std::log(ab / (1.0 - ab));
  };
  const stadi_step_t &st = sched[idx];
  const double h = lam(st.t_prev) - lam(st.t), hp = lam(st.t) - lam(sched[idx - 1].t);
  const double r = hp / h;
  *c1 = (float)(1.0 + 0.5 / r);
  *c2 = (float)(-0.5 / r);
}

// ---------------------------------------------------------------- kernel timing
// Wrap one launch of class `cls` in a pair of CUDA events on its stream when
// timing is enabled; `flops` / `bytes` are the launch's ALGORITHMIC work
// (DESIGN.md §6), accumulated beside the measured time.
template <typename F>
cudaError_t timed(stadi_ctx *ctx, int cls, double flops, double bytes, cudaStream_t s, F &&f) {
  if (!ctx->ktime) return f();
  auto &k = ctx->kt[cls];
  if (k.used == k.ev.size()) {
    cudaEvent_t a, b;
    cudaError_t e = cudaEventCreate(&a);
    if (e != cudaSuccess) return e;
    e = cudaEventCreate(&b);
    if (e != cudaSuccess) return e;
    k.ev.push_back({a, b});
  }
  auto &pr = k.ev[k.used++];
  cudaError_t e = cudaEventRecord(pr.first, s);
  if (e != cudaSuccess) return e;
  e = f();
  if (e != cudaSuccess) return e;
  k.launches += 1;
  k.flops += flops;
  k.bytes += bytes;
  return cudaEventRecord(pr.second, s);
}
// Fold the recorded event pairs into the per-class totals (caller synchronised).
cudaError_t collect_timing(stadi_ctx *ctx) {
  for (auto &k : ctx->kt) {
    for (size_t i = 0; i < k.used; ++i) {
      float ms = 0.f;
      cudaError_t e = cudaEventElapsedTime(&ms, k.ev[i].first, k.ev[i].second);
      if (e != cudaSuccess) return e;
      k.ms += ms;
    }
    k.used = 0;
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------- kernel dispatch
cudaError_t gemm(stadi_ctx *ctx, const void *A, const void *W, int M, int N, int K, int epi,
                 const EpiParams &ep, cudaStream_t s) {
  return timed(ctx, STADI_KCLASS_GEMM, 2.0 * M * N * K, 0.0, s, [&] {
    if (ctx->dtype == STADI_DTYPE_BF16) {
      EpiParams e2 = ep;
      e2.ws = ctx->splitk_ws;
      e2.ws_elems = ctx->splitk_elems;
      return tc_gemm_bf16((const bf16 *)A, (const bf16 *)W, M, N, K, epi, e2,
                          std::max(1, ctx->num_sms - ctx->emu_ctas), s);
    }
    return simt_gemm<float>((const float *)A, (const float *)W, M, N, K, epi, ep, s);
  });
}
cudaError_t attention(stadi_ctx *ctx, int cls, const void *q, const void *kv, void *o, int Nq,
                      int Nkv, cudaStream_t s) {
  const Dims &m = ctx->dm;
  const int B = ctx->Bf;
  const double flops = 4.0 * Nq * Nkv * m.hd * B * m.H;  // QK^T + PV, 2 flops per MAC
  return timed(ctx, cls, flops, 0.0, s, [&] {
    if (ctx->dtype == STADI_DTYPE_BF16)
      return tc_attention_bf16((const bf16 *)q, (const bf16 *)kv, (bf16 *)o, Nq, Nkv, B, m.H,
                               m.hd, s);
    return simt_attention<float>((const float *)q, (const float *)kv, (float *)o, Nq, Nkv, B,
                                 m.H, m.hd, s);
  });
}
cudaError_t lnmod(stadi_ctx *ctx, const float *x, void *y, int M, const float *shift,
                  const float *scale, int bs, int do_norm, cudaStream_t s) {
  const double bytes = (double)M * ctx->dm.d * (4 + ctx->esz);  // fp32 in, T out
  return timed(ctx, STADI_KCLASS_NORM, 0.0, bytes, s, [&] {
    if (ctx->dtype == STADI_DTYPE_BF16)
      return ln_modulate<bf16>(x, (bf16 *)y, M, ctx->dm.d, ctx->Bf, shift, scale, bs, do_norm,
                               s);
    return ln_modulate<float>(x, (float *)y, M, ctx->dm.d, ctx->Bf, shift, scale, bs, do_norm,
                              s);
  });
}

int widx(stadi_ctx *ctx, const std::string &name) {
  for (size_t i = 0; i < ctx->man.size(); ++i)
    if (ctx->man[i].name == name) return (int)i;
  return -1;
}
void *WT(stadi_ctx *ctx, const std::string &n) { return ctx->wT[widx(ctx, n)]; }
float *WF(stadi_ctx *ctx, const std::string &n) { return ctx->wf[widx(ctx, n)]; }

// Attention with an explicit head count (U-Net levels: d = C, hd = C / H).
cudaError_t attention_h(stadi_ctx *ctx, int cls, const void *q, const void *kv, void *o, int Nq,
                        int Nkv, int H, int C, cudaStream_t s) {
  const int B = ctx->dm.B, hd = C / H;
  const double flops = 4.0 * Nq * Nkv * hd * B * H;
  return timed(ctx, cls, flops, 0.0, s, [&] {
    if (ctx->dtype == STADI_DTYPE_BF16)
      return tc_attention_bf16((const bf16 *)q, (const bf16 *)kv, (bf16 *)o, Nq, Nkv, B, H, hd,
                               s);
    return simt_attention<float>((const float *)q, (const float *)kv, (float *)o, Nq, Nkv, B, H,
                                 hd, s);
  });
}

void free_graphs(stadi_ctx *ctx);

}  // namespace

#include "ipc.cuh"
#include "green.cuh"
#include "unet_exec.cuh"

namespace {

void free_graphs(stadi_ctx *ctx) {
  for (auto &g : ctx->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  ctx->graphs.clear();
}

void free_plan_buffers(stadi_ctx *ctx) {
  free_graphs(ctx);
  unet_free_plan(ctx);
  for (auto &r : ctx->ranks) {
    for (void *p : {(void *)r.x_band, (void *)r.x_res, r.xmod, r.q, r.o, r.h1, (void *)r.hist})
      pfree(ctx, p);
    if (!(ctx->ipc_mode && ctx->plan.cfg_split)) pfree(ctx, r.eps_raw);  // else in the arena
    if (!ctx->ipc_mode)  // IPC mode: the slots live in the (persistent) exchange arena
      for (void *p : r.kv) pfree(ctx, p);
  }
  ctx->ranks.clear();
  ctx->program.clear();
  for (auto e : ctx->ev_done) cudaEventDestroy(e);
  ctx->ev_done.clear();
  ctx->ev_used.clear();
  if (ctx->sub_comm && ctx->sub_comm != ctx->world_comm && nccl().CommDestroy)
    nccl().CommDestroy(ctx->sub_comm);
  ctx->sub_comm = nullptr;
  ctx->has_plan = false;
  ctx->begun = false;
}

int64_t slot_elems(const stadi_ctx *ctx) {
  const Dims &m = ctx->dm;
  return (int64_t)m.hp * m.wp * ctx->Bf * 2 * m.d;
}

}  // namespace

// ====================================================================== C ABI
extern "C" const char *stadi_last_error(const stadi_ctx *ctx) {
  return ctx ? ctx->err.c_str() : tls_error().c_str();
}

extern "C" stadi_status stadi_weight_count(const stadi_model_desc *desc, uint32_t *n) {
  if (!desc || !n) return fail(nullptr, STADI_EINVAL, "NULL argument");
  Dims d;
  std::string e;
  if (!make_dims(*desc, d, e)) return fail(nullptr, STADI_EINVAL, "%s", e.c_str());
  *n = (uint32_t)manifest(d).size();
  return STADI_OK;
}

extern "C" stadi_status stadi_weight_info(const stadi_model_desc *desc, uint32_t index,
                                          char *name_buf, uint32_t name_cap, uint64_t *numel) {
  if (!desc) return fail(nullptr, STADI_EINVAL, "NULL argument");
  Dims d;
  std::string e;
  if (!make_dims(*desc, d, e)) return fail(nullptr, STADI_EINVAL, "%s", e.c_str());
  auto man = manifest(d);
  if (index >= man.size()) return fail(nullptr, STADI_EINVAL, "index out of range");
  if (name_buf && name_cap) {
    std::strncpy(name_buf, man[index].name.c_str(), name_cap - 1);
    name_buf[name_cap - 1] = 0;
  }
  if (numel) *numel = (uint64_t)(man[index].rows * man[index].cols);
  return STADI_OK;
}

extern "C" stadi_status stadi_ipc_session_id(uint8_t out[128]) {
  if (!out) return fail(nullptr, STADI_EINVAL, "NULL argument");
  std::memset(out, 0, 128);
  FILE *f = std::fopen("/dev/urandom", "rb");
  size_t n = f ? std::fread(out, 1, 16, f) : 0;
  if (f) std::fclose(f);
  if (n != 16) {  // no urandom: pid + clock
    const uint64_t a = (uint64_t)getpid(), b = (uint64_t)std::chrono::steady_clock::now()
                                                   .time_since_epoch().count();
    std::memcpy(out, &a, 8);
    std::memcpy(out + 8, &b, 8);
  }
  return STADI_OK;
}

extern "C" stadi_status stadi_nccl_unique_id(uint8_t out[128]) {
  if (!out) return fail(nullptr, STADI_EINVAL, "NULL argument");
  if (!nccl().ok) return fail(nullptr, STADI_ENCCL, "libnccl.so.2 not loadable");
  ncclUniqueId id;
  ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, STADI_ENCCL, "ncclGetUniqueId failed");
  std::memcpy(out, &id, 128);
  return STADI_OK;
}

extern "C" stadi_status stadi_create(const stadi_model_desc *model, const stadi_dist_desc *dist,
                                     stadi_ctx **out) {
  if (!model || !dist || !out) return fail(nullptr, STADI_EINVAL, "NULL argument");
  *out = nullptr;
  Dims dm;
  std::string e;
  if (!make_dims(*model, dm, e)) return fail(nullptr, STADI_EINVAL, "%s", e.c_str());
  if (model->dtype != STADI_DTYPE_BF16 && model->dtype != STADI_DTYPE_FP32_DEBUG)
    return fail(nullptr, STADI_EINVAL, "bad dtype");
  if (model->sampler != STADI_SAMPLER_DDIM && model->sampler != STADI_SAMPLER_DDPM &&
      model->sampler != STADI_SAMPLER_DPM2M)
    return fail(nullptr, STADI_EINVAL, "bad sampler");
  if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world || dist->n_local < 1 ||
      (dist->world > 1 && dist->n_local != 1) || dist->world * dist->n_local > STADI_MAX_GPUS)
    return fail(nullptr, STADI_EINVAL, "bad dist desc (n_local > 1 requires world == 1)");
  if (model->dtype == STADI_DTYPE_BF16) {
    if (!dm.unet && !tc_attention_supported(dm.hd))
      return fail(nullptr, STADI_EUNSUPPORTED, "head dim %d not supported by the tcgen05 kernel",
                  dm.hd);
    for (int l = 0; dm.unet && l < dm.levels(); ++l)
      if ((dm.tdepth[l] || (l == dm.levels() - 1 && dm.mid_depth)) &&
          !tc_attention_supported(dm.ch[l] / dm.heads[l]))
        return fail(nullptr, STADI_EUNSUPPORTED, "head dim %d not supported by the tcgen05 kernel",
                    dm.ch[l] / dm.heads[l]);
  }
  auto ctx = std::make_unique<stadi_ctx>();
  ctx->dm = dm;
  ctx->dtype = model->dtype;
  ctx->sampler = model->sampler;
  ctx->esz = model->dtype == STADI_DTYPE_BF16 ? 2 : 4;
  ctx->device = dist->device;
  ctx->rank = dist->rank;
  ctx->world = dist->world;
  ctx->n_local = dist->n_local;
  ctx->G = dist->world * dist->n_local;
  if (dist->world > 1 && dist->transport != STADI_TRANSPORT_NCCL &&
      dist->transport != STADI_TRANSPORT_IPC)
    return fail(nullptr, STADI_EINVAL, "bad transport");
  {
    const char *fe = getenv("STADI_FORCE_NCCL");
    ctx->ipc_mode = dist->world > 1 && dist->transport == STADI_TRANSPORT_IPC;
    ctx->nccl = (dist->world > 1 && !ctx->ipc_mode) ||
                (dist->world == 1 && dist->n_local == 1 && fe && fe[0] == '1');
  }
  ctx->man = manifest(dm);
  ctx->fin_ld = (int)rup(dm.p * dm.p * dm.c_out, 64);
  alpha_bar(dm.schedule_linear != 0, ctx->abar);
  stadi_ctx *c = ctx.get();
  {
    stadi_ctx *ctx = c;  // for CK
    CK(cudaSetDevice(dist->device));
    CK(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dist->device));
    int lo, hi;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    if (dist->vgpu_sms > 0) {  // virtual GPU: an SM partition of the device (green.cuh)
      if (dist->n_local != 1) return ctx_fail(ctx, STADI_EINVAL, "vgpu_sms needs n_local == 1");
      ST(green_init(ctx, dist->rank, dist->vgpu_sms, hi));
    } else {
      CK(cudaStreamCreateWithPriority(&ctx->comm, cudaStreamNonBlocking, hi));
      CK(cudaStreamCreateWithFlags(&ctx->astream, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking));
    }
    CK(cudaEventCreateWithFlags(&ctx->ev_ready, cudaEventDisableTiming));
    // positional embedding of the full token grid, fp64 on the host (pins the
    // values to 1 ulp of fp32), [sin(c w), cos(c w), sin(r w), cos(r w)]
    const int q4 = dm.d / 4;
    std::vector<float> pos((size_t)dm.hp * dm.wp * dm.d);
    for (int r = 0; r < dm.hp; ++r)
      for (int cc = 0; cc < dm.wp; ++cc) {
        float *row = &pos[((size_t)r * dm.wp + cc) * dm.d];
        for (int k = 0; k < q4; ++k) {
          const double w = 1.0 / std::pow(10000.0, (double)k / q4);
          row[k] = (float)std::sin(cc * w);
          row[q4 + k] = (float)std::cos(cc * w);
          row[2 * q4 + k] = (float)std::sin(r * w);
          row[3 * q4 + k] = (float)std::cos(r * w);
        }
      }
    CK(dalloc(ctx, &ctx->pos_full, pos.size() * 4));
    CK(cudaMemcpy(ctx->pos_full, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice));
    if (ctx->dtype == STADI_DTYPE_BF16) {
      // split-K uses at most (#SMs) partial tiles of 128 x 256 fp32: 19 MB on B200
      ctx->splitk_elems = (long)ctx->num_sms * 128 * 256;
      CK(dalloc(ctx, &ctx->splitk_ws, (size_t)ctx->splitk_elems * 4));
    }
    if (ctx->nccl) {
      if (!nccl().ok) return ctx_fail(ctx, STADI_ENCCL, "libnccl.so.2 not loadable");
      ncclUniqueId id;
      if (dist->world == 1) {
        CKN(nccl().GetUniqueId(&id));
      } else {
        if (!dist->nccl_id) return ctx_fail(ctx, STADI_EINVAL, "nccl_id required when world > 1");
        std::memcpy(&id, dist->nccl_id, 128);
      }
      CKN(nccl().CommInitRank(&ctx->world_comm, dist->world, id, dist->rank));
      // Launch every collective this context uses once now (grouped broadcasts of
      // bf16 / fp32 rows, small and large, and the fp64 all-gather of the
      // profiler), so that NCCL's kernels are loaded before the occupancy emulator
      // can be resident: CUDA lazy loading of a kernel first launched under a
      // resident kernel may need a context synchronisation -> deadlock (observed).
      {
        const size_t big = (size_t)8 << 20;
        void *buf = nullptr;
        CK(cudaMalloc(&buf, big * 4 + 64 * dist->world));
        CK(cudaMemset(buf, 0, big * 4 + 64 * dist->world));
        for (size_t n : {(size_t)256, big}) {
          for (ncclDataType_t dt : {ncclBfloat16, ncclFloat32}) {
            CKN(nccl().GroupStart());
            const size_t seg = n / dist->world;  // disjoint per-root segments
            for (int r = 0; r < dist->world; ++r) {
              void *p = (char *)buf + r * seg * 4;
              CKN(nccl().Broadcast(p, p, seg, dt, r, ctx->world_comm, ctx->comm));
            }
            CKN(nccl().GroupEnd());
          }
        }
        double *d64 = reinterpret_cast<double *>((char *)buf + big * 4);
        CKN(nccl().AllGather(d64, d64 + 1, 1, ncclFloat64, ctx->world_comm, ctx->comm));
        CK(cudaStreamSynchronize(ctx->comm));
        CK(cudaFree(buf));
      }
    }
    if (ctx->ipc_mode) {
      if (!dist->nccl_id) return ctx_fail(ctx, STADI_EINVAL, "IPC transport needs a session id");
      if (!memops().ok)
        return ctx_fail(ctx, STADI_EUNSUPPORTED, "stream memory operations unavailable");
      ctx->ipc = std::make_unique<IpcState>();
      IpcState &I = *ctx->ipc;
      I.session = hexs(dist->nccl_id, 16);
      struct stat sb;
      I.dir = (stat("/dev/shm", &sb) == 0 && access("/dev/shm", W_OK) == 0) ? "/dev/shm" : "/tmp";
      CK(dalloc(ctx, &I.probe, 256));
      CK(cudaMemset(I.probe, 0, 256));
      I.graphs_ok = ipc_probe_graphs(ctx);
    }
    {  // pinned staging: noise + result + text + pooled + time features + small items
      const size_t lat = (size_t)dm.lat_h * dm.lat_w * dm.c_in * 4;
      const size_t txt = (size_t)dm.B * dm.txt_len * dm.txt_dim * 4;
      const size_t tf = (size_t)1000 * std::max(256, dm.unet ? dm.ch[0] : 256) * 4;
      ctx->stage_cap = 2 * lat + txt + (size_t)dm.B * (dm.pooled_dim + 6 * 256 + 64) * 4 + tf +
                       (64 << 10);
      CK(cudaMallocHost(&ctx->stage, ctx->stage_cap));
      CK(cudaEventCreateWithFlags(&ctx->stage_ev, cudaEventDisableTiming));
    }
    CK(dalloc(ctx, &ctx->seed_dev, 8));
    CK(cudaMemset(ctx->seed_dev, 0, 8));
    CK(cudaMalloc(&ctx->emu_flag_dev, 64));
    CK(cudaMemset(ctx->emu_flag_dev, 0, 64));
    if (!ctx->green_ctx) {
      CK(cudaStreamCreateWithFlags(&ctx->emu_stream, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&ctx->emu_ctl, cudaStreamNonBlocking));
    }
  }
  *out = ctx.release();
  return STADI_OK;
}

extern "C" void stadi_destroy(stadi_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->emu_ctas) {
    cudaMemsetAsync(ctx->emu_flag_dev, 1, 4, ctx->emu_ctl);
    cudaStreamSynchronize(ctx->emu_stream);
  }
  cudaDeviceSynchronize();
  free_plan_buffers(ctx);
  ipc_release(ctx);
  for (void *p : ctx->allocs) cudaFree(p);
  for (void *p : ctx->wT) cudaFree(p);
  for (float *p : ctx->wf) cudaFree(p);
  if (ctx->world_comm && nccl().CommDestroy) nccl().CommDestroy(ctx->world_comm);
  if (ctx->comm) cudaStreamDestroy(ctx->comm);
  if (ctx->astream) cudaStreamDestroy(ctx->astream);
  if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
  if (ctx->emu_stream) cudaStreamDestroy(ctx->emu_stream);
  if (ctx->emu_ctl) cudaStreamDestroy(ctx->emu_ctl);
  if (ctx->wstream) cudaStreamDestroy(ctx->wstream);
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->stage_ev) cudaEventDestroy(ctx->stage_ev);
  if (ctx->stage) cudaFreeHost(ctx->stage);
  if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
  if (ctx->green_ctx && green_api().GreenCtxDestroy) green_api().GreenCtxDestroy(ctx->green_ctx);
  if (ctx->ev_ready) cudaEventDestroy(ctx->ev_ready);
  for (auto &k : ctx->kt)
    for (auto &pr : k.ev) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  if (ctx->emu_flag_dev) cudaFree(ctx->emu_flag_dev);
  cudaGetLastError();
  delete ctx;
}

namespace {
// fp32 -> T conversion on the device (bf16: round-to-nearest-even)
cudaError_t upload_T(stadi_ctx *ctx, const float *host, int64_t n, void **dst_T, float **dst_f) {
  float *f = nullptr;
  cudaError_t e = cudaMalloc(&f, n * 4);
  if (e != cudaSuccess) return e;
  e = cudaMemcpy(f, host, n * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return e;
  if (ctx->dtype == STADI_DTYPE_BF16) {
    bf16 *t = nullptr;
    e = cudaMalloc(&t, n * 2);
    if (e != cudaSuccess) return e;
    e = cast_f32<bf16>(f, t, n, 0);
    if (e != cudaSuccess) return e;
    // fp32 copy holds the bf16-rounded values (the oracle's bf16 parity weights)
    std::vector<float> tmp;
    (void)tmp;
    if (dst_T) *dst_T = t;
    else cudaFree(t);
  } else if (dst_T) {
    *dst_T = f;
  }
  *dst_f = f;
  return cudaSuccess;
}

__global__ void round_bf16_inplace(float *x, long n) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = __bfloat162float(__float2bfloat16_rn(x[i]));
}
}  // namespace

extern "C" stadi_status stadi_load_weights(stadi_ctx *ctx, uint32_t n_tensors,
                                           const float *const *host, const uint64_t *numels) {
  ALIVE();
  if (!host || !numels) return ctx_fail(ctx, STADI_EINVAL, "NULL argument");
  if (n_tensors != ctx->man.size())
    return ctx_fail(ctx, STADI_EINVAL, "expected %zu tensors, got %u", ctx->man.size(), n_tensors);
  for (uint32_t i = 0; i < n_tensors; ++i) {
    const uint64_t want = (uint64_t)(ctx->man[i].rows * ctx->man[i].cols);
    if (numels[i] != want || !host[i])
      return ctx_fail(ctx, STADI_EINVAL, "tensor %u (%s): numel %llu, expected %llu", i,
                      ctx->man[i].name.c_str(), (unsigned long long)numels[i],
                      (unsigned long long)want);
  }
  CK(cudaSetDevice(ctx->device));
  if (ctx->weights_loaded) return ctx_fail(ctx, STADI_ESTATE, "weights already loaded");
  const Dims &m = ctx->dm;
  const bool bf = ctx->dtype == STADI_DTYPE_BF16;
  if (m.unet) {
    ST(unet_load_weights(ctx, host));
    CK(cudaStreamSynchronize(0));
    ctx->weights_loaded = true;
    return STADI_OK;
  }
  ctx->wT.assign(n_tensors, nullptr);
  ctx->wf.assign(n_tensors, nullptr);
  for (uint32_t i = 0; i < n_tensors; ++i) {
    const auto &ts = ctx->man[i];
    const int64_t n = ts.rows * ts.cols;
    CK(upload_T(ctx, host[i], n, ts.gemm_weight ? &ctx->wT[i] : nullptr, &ctx->wf[i]));
    if (bf) {
      round_bf16_inplace<<<(unsigned)((n + 255) / 256), 256>>>(ctx->wf[i], n);
      CK(cudaGetLastError());
    }
  }
  // contiguous per-block tensors for the batched conditioning GEMM
  const int64_t d = m.d;
  if (!m.text) {
    CK(dalloc(ctx, &ctx->ada_all, m.depth * 6 * d * d * ctx->esz));
    CK(dalloc(ctx, &ctx->ada_all_b, m.depth * 6 * d * 4));
    for (int l = 0; l < m.depth; ++l) {
      const std::string p = "blocks." + std::to_string(l) + ".";
      CK(cudaMemcpy((char *)ctx->ada_all + l * 6 * d * d * ctx->esz, WT(ctx, p + "ada.w"),
                    6 * d * d * ctx->esz, cudaMemcpyDeviceToDevice));
      CK(cudaMemcpy(ctx->ada_all_b + l * 6 * d, WF(ctx, p + "ada.b"), 6 * d * 4,
                    cudaMemcpyDeviceToDevice));
    }
  } else {
    CK(dalloc(ctx, &ctx->sst_all, m.depth * 6 * d * 4));
    for (int l = 0; l < m.depth; ++l)
      CK(cudaMemcpy(ctx->sst_all + l * 6 * d, WF(ctx, "blocks." + std::to_string(l) + ".sst"),
                    6 * d * 4, cudaMemcpyDeviceToDevice));
  }
  // final linear, rows zero-padded to fin_ld (tcgen05 N granularity)
  const int nf = m.p * m.p * m.c_out;
  CK(dalloc(ctx, &ctx->final_w, (size_t)ctx->fin_ld * d * ctx->esz));
  CK(cudaMemset(ctx->final_w, 0, (size_t)ctx->fin_ld * d * ctx->esz));
  CK(cudaMemcpy(ctx->final_w, WT(ctx, "final.linear.w"), (size_t)nf * d * ctx->esz,
                cudaMemcpyDeviceToDevice));
  CK(dalloc(ctx, &ctx->final_b, ctx->fin_ld * 4));
  CK(cudaMemset(ctx->final_b, 0, ctx->fin_ld * 4));
  CK(cudaMemcpy(ctx->final_b, WF(ctx, "final.linear.b"), nf * 4, cudaMemcpyDeviceToDevice));
  CK(cudaStreamSynchronize(0));
  ctx->weights_loaded = true;
  return STADI_OK;
}

// ---------------------------------------------------------------- plan install
extern "C" stadi_status stadi_set_plan(stadi_ctx *ctx, const stadi_plan_t *plan) {
  ALIVE();
  if (!plan) return ctx_fail(ctx, STADI_EINVAL, "NULL plan");
  const Dims &m = ctx->dm;
  if ((int)plan->n_gpus != ctx->G)
    return ctx_fail(ctx, STADI_EINVAL, "plan has %u GPUs, group has %d", plan->n_gpus, ctx->G);
  const uint32_t unit = m.unet ? (1u << (m.levels() - 1)) : (uint32_t)m.p;
  if ((int64_t)plan->p_total * plan->rows_per_unit != m.lat_h || plan->rows_per_unit % unit)
    return ctx_fail(ctx, STADI_EINVAL,
                    "plan covers %u x %u rows; latent has %d rows (unit must be a multiple of "
                    "%u rows, R6)",
                    plan->p_total, plan->rows_per_unit, m.lat_h, unit);
  if (plan->m_base > 1000) return ctx_fail(ctx, STADI_EINVAL, "M_base > 1000");
  CK(cudaSetDevice(ctx->device));
  DBG("set_plan: quiesce");
  CK(quiesce(ctx));
  DBG("set_plan: quiesced");
  free_plan_buffers(ctx);
  if (plan->cfg_split && (m.unet || m.B != 2 || ctx->nccl))
    return ctx_fail(ctx, STADI_EUNSUPPORTED,
                    "CFG batch split (R33) needs a DiT-family model with CFG, local / IPC mode");
  ctx->plan = *plan;
  ctx->Bf = plan->cfg_split ? 1 : m.B;
  const int g0 = ctx->rank * ctx->n_local;
  for (int k = 0; k < ctx->n_local; ++k) {
    const int g = g0 + k;
    if (plan->tier[g] == 0) continue;  // excluded (Eq. 4 third case)
    Rank r;
    r.g = g;
    r.tier = plan->tier[g];
    r.row_begin = (int)plan->row_begin[g];
    r.rows = (int)plan->rows[g];
    r.tok_begin = r.row_begin / m.p * m.wp;
    r.n_tok = r.rows / m.p * m.wp;
    r.branch = plan->cfg_split ? plan->branch[g] : 0;
    r.partner = plan->cfg_split ? plan->partner[g] : -1;
    uint32_t n = 0;
    if (stadi_schedule(plan, g, nullptr, 0, &n) != STADI_OK)
      return ctx_fail(ctx, STADI_EINVAL, "bad plan: %s", tls_error().c_str());
    r.sched.resize(n);
    stadi_schedule(plan, g, r.sched.data(), n, &n);
    const int64_t M = (int64_t)r.n_tok * ctx->Bf;
    CK(pmalloc(ctx, &r.x_band, std::max<int64_t>(16, (int64_t)r.rows * m.lat_w * m.c_in * 4)));
    if (ctx->sampler == STADI_SAMPLER_DPM2M)
      CK(pmalloc(ctx, &r.hist, std::max<int64_t>(16, (int64_t)r.rows * m.lat_w * m.c_in * 4)));
    if (m.unet) {  // the U-Net program owns its buffers (unet_set_plan)
      ctx->ranks.push_back(std::move(r));
      continue;
    }
    CK(pmalloc(ctx, &r.x_res, std::max<int64_t>(16, M * m.d * 4)));
    CK(pmalloc(ctx, &r.xmod, std::max<int64_t>(16, M * m.d * ctx->esz)));
    CK(pmalloc(ctx, &r.q, std::max<int64_t>(16, M * m.d * ctx->esz)));
    CK(pmalloc(ctx, &r.o, std::max<int64_t>(16, M * m.d * ctx->esz)));
    CK(pmalloc(ctx, &r.h1, std::max<int64_t>(16, M * 4 * m.d * ctx->esz)));
    // eps of both CFG rows [n_tok, B, fin_ld]: under the CFG split the rank writes its
    // branch's columns, the partner's arrive by the pair exchange (IPC: in the arena)
    if (!(ctx->ipc_mode && plan->cfg_split))
      CK(pmalloc(ctx, &r.eps_raw, std::max<int64_t>(16, (int64_t)r.n_tok * m.B * ctx->fin_ld * 4)));
    r.kv.assign(m.depth * 2, nullptr);
    CK(cudaStreamSynchronize(ctx->astream));
    if (!ctx->ipc_mode) {
      for (auto &p : r.kv) {
        CK(pmalloc(ctx, &p, slot_elems(ctx) * ctx->esz));
        CK(cudaMemsetAsync(p, 0, slot_elems(ctx) * ctx->esz, ctx->astream));
      }
    }
    CK(cudaStreamSynchronize(ctx->astream));
    ctx->ranks.push_back(std::move(r));
  }
  // program
  if (ctx->nccl || ctx->ipc_mode) {
    if (!ctx->ranks.empty())
      for (size_t k = 0; k < ctx->ranks[0].sched.size(); ++k)
        ctx->program.push_back({Part{0, ctx->ranks[0].sched[k], (int)k}});
  } else {
    for (int mm = 0; mm < (int)plan->m_base; ++mm) {
      std::vector<Part> ph;
      for (int li = 0; li < (int)ctx->ranks.size(); ++li)
        for (size_t k = 0; k < ctx->ranks[li].sched.size(); ++k)
          if (ctx->ranks[li].sched[k].m == mm) ph.push_back(Part{li, ctx->ranks[li].sched[k], (int)k});
      if (!ph.empty()) ctx->program.push_back(ph);
    }
  }
  // NCCL: communicator over the included ranks + exchange events
  if (ctx->nccl) {
    const bool inc = !ctx->ranks.empty();
    bool all_inc = true;
    for (uint32_t i = 0; i < plan->n_gpus; ++i) all_inc &= plan->tier[i] != 0;
    if (all_inc) {
      ctx->sub_comm = ctx->world_comm;
    } else {
      if (!nccl().CommSplit) return ctx_fail(ctx, STADI_ENCCL, "ncclCommSplit unavailable");
      CKN(nccl().CommSplit(ctx->world_comm, inc ? 0 : NCCL_SPLIT_NOCOLOR, ctx->rank,
                           &ctx->sub_comm, nullptr));
    }
    ctx->ev_done.assign(m.depth * 2, nullptr);
    ctx->ev_used.assign(m.depth * 2, 0);
    for (auto &e : ctx->ev_done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (m.unet) {
    ST(unet_set_plan(ctx));
  } else if (ctx->ipc_mode) {  // K/V slots of every site and parity in the IPC arena
    ipc_layout_begin(ctx);
    IpcState &I = *ctx->ipc;
    for (int l = 0; l < m.depth; ++l)
      for (int par = 0; par < 2; ++par)
        I.site_off[par].push_back(ipc_reserve(ctx, slot_elems(ctx) * ctx->esz));
    int n_sites = m.depth;
    if (plan->cfg_split) {  // site `depth`: the pair's eps exchange [tokens, 2, fin_ld] f32
      const size_t eb = (size_t)m.hp * m.wp * 2 * ctx->fin_ld * 4;
      I.site_off[0].push_back(ipc_reserve(ctx, eb));
      I.site_off[1].push_back(I.site_off[0].back());
      ++n_sites;
    }
    ST(ipc_commit(ctx, n_sites));
    for (auto &r : ctx->ranks) {
      for (int l = 0; l < m.depth; ++l)
        for (int par = 0; par < 2; ++par) r.kv[l * 2 + par] = I.arena + I.site_off[par][l];
      if (plan->cfg_split) r.eps_raw = (float *)(I.arena + I.site_off[0][m.depth]);
    }
  }
  ctx->has_plan = true;
  return STADI_OK;
}

// ---------------------------------------------------------------- request begin
namespace {
stadi_status begin_impl(stadi_ctx *ctx, const float *noise_full, const stadi_cond *cond,
                        void *stream);
stadi_status gather_impl(stadi_ctx *ctx, float *out_full, void *stream);
stadi_status run_phase(stadi_ctx *ctx, const std::vector<Part> &phase, cudaStream_t s);
}  // namespace

// Public entry points: (virtual GPU) the work runs on the context's green stream,
// joined after / before the caller's stream.
extern "C" stadi_status stadi_begin(stadi_ctx *ctx, const float *noise_full,
                                    const stadi_cond *cond, void *stream) {
  ALIVE();
  NvtxRange nv("stadi_begin");
  cudaStream_t w;
  CK(enter_stream(ctx, (cudaStream_t)stream, &w));
  ST(begin_impl(ctx, noise_full, cond, w));
  CK(leave_stream(ctx, (cudaStream_t)stream));
  return STADI_OK;
}
extern "C" stadi_status stadi_gather(stadi_ctx *ctx, float *out_full, void *stream) {
  ALIVE();
  NvtxRange nv("stadi_gather");
  cudaStream_t w;
  CK(enter_stream(ctx, (cudaStream_t)stream, &w));
  ST(gather_impl(ctx, out_full, w));
  CK(leave_stream(ctx, (cudaStream_t)stream));
  return STADI_OK;
}

namespace {
stadi_status begin_impl(stadi_ctx *ctx, const float *noise_full, const stadi_cond *cond,
                        void *stream) {
  ALIVE();
  if (!ctx->has_plan) return ctx_fail(ctx, STADI_ESTATE, "stadi_begin before stadi_set_plan");
  if (!ctx->weights_loaded) return ctx_fail(ctx, STADI_ESTATE, "weights not loaded");
  if (!noise_full || !cond) return ctx_fail(ctx, STADI_EINVAL, "NULL argument");
  const Dims &m = ctx->dm;
  if (m.text ? !cond->text : !cond->labels)
    return ctx_fail(ctx, STADI_EINVAL, "conditioning missing (%s)", m.text ? "text" : "labels");
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(ctx->device));
  ctx->ddpm_seed = cond->ddpm_seed;
  CK(stage_reset(ctx));
  // the sampler reads the key from device memory (graph replays see this request's seed)
  CK(cudaMemcpyAsync(ctx->seed_dev, stage_h2d(ctx, &ctx->ddpm_seed, 8), 8,
                     cudaMemcpyHostToDevice, s));
  // Tail of the call, after the conditioning: (IPC, first request of a plan) one
  // compute-only probe step that loads every kernel of the path -- CUDA lazy loading of
  // a kernel first launched while this process has a stream blocked in an exchange wait
  // can need a context synchronisation that never completes (the flag comes from a
  // peer that waits for us); then the noise bands and the flag barrier.
  auto finish = [&]() -> stadi_status {
    if (ctx->ipc_mode && !ctx->kernels_warm && !ctx->ranks.empty() && !ctx->program.empty()) {
      ctx->probe = true;
      const stadi_status st = run_phase(ctx, {ctx->program[0][0]}, s);
      ctx->probe = false;
      ST(st);
      CK(cudaStreamSynchronize(s));
      ctx->kernels_warm = true;
      DBG("begin: kernels loaded");
    }
    const bool dev = is_device_ptr(noise_full);
    const size_t row_bytes = (size_t)m.lat_w * m.c_in * 4;
    for (auto &r : ctx->ranks) {  // noise bands (overwrite the probe's band)
      const float *src = noise_full + (size_t)r.row_begin * m.lat_w * m.c_in;
      const void *st = dev ? src : stage_h2d(ctx, src, row_bytes * r.rows);
      if (!st) return ctx_fail(ctx, STADI_ENOMEM, "host staging exhausted");
      CK(cudaMemcpyAsync(r.x_band, st, row_bytes * r.rows,
                         dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    }
    DBG("begin: noise copied");
    if (ctx->ipc_mode) ST(ipc_begin(ctx, s));  // flag reset + device-side barrier
    DBG("begin: barrier enqueued");
    CK(cudaEventRecord(ctx->stage_ev, s));
    ctx->stage_pending = true;
    ctx->begun = true;
    ctx->exch_bytes = 0;
    return STADI_OK;
  };
  // ---- conditioning for every fast-grid timestep (one batched GEMM each)
  const int nt = (int)ctx->plan.m_base;
  const int64_t d = m.d;
  const int B = m.B;
  if (!m.unet && ctx->cond_cap_nt < (size_t)nt) {
    // (re)allocate per-request conditioning buffers
    CK(quiesce(ctx));
    for (void *p : {(void *)ctx->mod, (void *)ctx->fmod, (void *)ctx->temb, (void *)ctx->tmp_f,
                    (void *)ctx->tfreq, ctx->csilu})
      pfree(ctx, p);
    CK(pmalloc(ctx, &ctx->mod, (size_t)nt * B * m.depth * 6 * d * 4));
    CK(pmalloc(ctx, &ctx->fmod, (size_t)nt * B * 2 * d * 4));
    CK(pmalloc(ctx, &ctx->temb, (size_t)nt * d * 4));
    CK(pmalloc(ctx, &ctx->tmp_f, (size_t)nt * 6 * d * 4));
    CK(pmalloc(ctx, &ctx->tfreq, (size_t)nt * 256 * 4));
    CK(pmalloc(ctx, &ctx->csilu, (size_t)nt * B * d * ctx->esz));
    CK(cudaStreamSynchronize(ctx->astream));
    ctx->cond_cap_nt = nt;
    free_graphs(ctx);  // captured steps reference the old conditioning buffers
    ctx->tfreq_nt = 0;
  }
  ctx->n_t = nt;
  if (m.unet) {
    ST(unet_begin(ctx, cond, s));
    return finish();
  }
  if (ctx->tfreq_nt != nt) {
    // sinusoidal timestep features of the fast grid, fp64 on the host (DiT
    // TimestepEmbedder); depends only on M_base, uploaded once per plan size
    std::vector<float> tf((size_t)nt * 256);
    const int ratio = 1000 / nt;
    for (int i = 0; i < nt; ++i) {
      const double t = ratio * (nt - 1 - i) + 1;  // fast grid (R18)
      for (int k = 0; k < 128; ++k) {
        const double f = std::exp(-std::log(10000.0) * k / 128.0);
        tf[(size_t)i * 256 + k] = (float)std::cos(t * f);
        tf[(size_t)i * 256 + 128 + k] = (float)std::sin(t * f);
      }
    }
    const void *st = stage_h2d(ctx, tf.data(), tf.size() * 4);
    if (!st) return ctx_fail(ctx, STADI_ENOMEM, "host staging exhausted");
    CK(cudaMemcpyAsync(ctx->tfreq, st, tf.size() * 4, cudaMemcpyHostToDevice, s));
    ctx->tfreq_nt = nt;
  }
  EpiParams ep{};
  ep.B = 1;
  ep.bias = WF(ctx, "t_embed.b1");
  ep.out = ctx->tmp_f;
  ep.ldo = (int)d;
  CK(simt_gemm<float>(ctx->tfreq, WF(ctx, "t_embed.w1"), nt, (int)d, 256, EPI_F32, ep, s));
  CK(silu_inplace(ctx->tmp_f, (long)nt * d, s));
  ep.bias = WF(ctx, "t_embed.b2");
  ep.out = ctx->temb;
  CK(simt_gemm<float>(ctx->tmp_f, WF(ctx, "t_embed.w2"), nt, (int)d, (int)d, EPI_F32, ep, s));
  if (!m.text) {
    if (!ctx->labels_dev) CK(dalloc(ctx, &ctx->labels_dev, 64 * 4));
    for (int b = 0; b < B; ++b)
      if (cond->labels[b] < 0 || cond->labels[b] > m.num_classes)
        return ctx_fail(ctx, STADI_EINVAL, "class label out of range");
    CK(cudaMemcpyAsync(ctx->labels_dev, stage_h2d(ctx, cond->labels, B * 4), B * 4,
                       cudaMemcpyHostToDevice, s));
    if (ctx->dtype == STADI_DTYPE_BF16)
      CK(class_cond<bf16>(ctx->temb, WF(ctx, "y_embed.table"), ctx->labels_dev, nt, B, (int)d,
                          (bf16 *)ctx->csilu, s));
    else
      CK(class_cond<float>(ctx->temb, WF(ctx, "y_embed.table"), ctx->labels_dev, nt, B, (int)d,
                           (float *)ctx->csilu, s));
    // adaLN for all blocks and all timesteps: [nt*B, d] x [depth*6d, d]^T
    ep.bias = ctx->ada_all_b;
    ep.out = ctx->mod;
    ep.ldo = (int)(m.depth * 6 * d);
    CK(gemm(ctx, ctx->csilu, ctx->ada_all, nt * B, (int)(m.depth * 6 * d), (int)d, EPI_F32, ep,
            s));
    ep.bias = WF(ctx, "final.ada.b");
    ep.out = ctx->fmod;
    ep.ldo = (int)(2 * d);
    CK(gemm(ctx, ctx->csilu, WT(ctx, "final.ada.w"), nt * B, (int)(2 * d), (int)d, EPI_F32, ep,
            s));
  } else {
    // adaLN-single: t0 = W SiLU(t_emb) + b ; mod_l = sst_l + t0 ; final = sst_f + t_emb
    if (ctx->dtype == STADI_DTYPE_BF16)
      CK(silu_cast<bf16>(ctx->temb, (bf16 *)ctx->csilu, (long)nt * d, s));
    else
      CK(silu_cast<float>(ctx->temb, (float *)ctx->csilu, (long)nt * d, s));
    ep.bias = WF(ctx, "t_block.b");
    ep.out = ctx->tmp_f;
    ep.ldo = (int)(6 * d);
    CK(gemm(ctx, ctx->csilu, WT(ctx, "t_block.w"), nt, (int)(6 * d), (int)d, EPI_F32, ep, s));
    CK(pixart_mods(ctx->tmp_f, ctx->temb, ctx->sst_all, WF(ctx, "final.sst"), nt, B, m.depth,
                   (int)d, ctx->mod, ctx->fmod, s));
    // caption projection + per-block cross-attention K/V (once per request)
    const int L = m.txt_len, Dt = m.txt_dim;
    const int64_t Mt = (int64_t)L * B;
    if (!ctx->text_T) {
      CK(dalloc(ctx, &ctx->text_T, Mt * Dt * ctx->esz));
      CK(dalloc(ctx, &ctx->y1, Mt * d * ctx->esz));
      CK(dalloc(ctx, &ctx->y, Mt * d * ctx->esz));
      ctx->kv_text.assign(m.depth, nullptr);
      for (auto &p : ctx->kv_text) CK(dalloc(ctx, &p, Mt * 2 * d * ctx->esz));
    }
    // [B, L, D] -> [L, B, D] (token-major, batch innermost) by strided copies;
    // text may be a host or a device pointer (cudaMemcpyDefault)
    if (!ctx->text_f) CK(dalloc(ctx, &ctx->text_f, Mt * Dt * 4));
    const float *txt = (const float *)stage_h2d(ctx, cond->text, (size_t)Mt * Dt * 4);
    if (!txt) return ctx_fail(ctx, STADI_ENOMEM, "host staging exhausted");
    for (int b = 0; b < B; ++b)
      CK(cudaMemcpy2DAsync(ctx->text_f + (size_t)b * Dt, (size_t)B * Dt * 4,
                           txt + (size_t)b * L * Dt, (size_t)Dt * 4, (size_t)Dt * 4, L,
                           cudaMemcpyDefault, s));
    if (ctx->dtype == STADI_DTYPE_BF16)
      CK(cast_f32<bf16>(ctx->text_f, (bf16 *)ctx->text_T, (long)(Mt * Dt), s));
    else
      CK(cudaMemcpyAsync(ctx->text_T, ctx->text_f, Mt * Dt * 4, cudaMemcpyDeviceToDevice, s));
    ep.bias = WF(ctx, "caption.b1");
    ep.out = ctx->y1;
    ep.ldo = (int)d;
    CK(gemm(ctx, ctx->text_T, WT(ctx, "caption.w1"), (int)Mt, (int)d, Dt, EPI_GELU, ep, s));
    ep.bias = WF(ctx, "caption.b2");
    ep.out = ctx->y;
    CK(gemm(ctx, ctx->y1, WT(ctx, "caption.w2"), (int)Mt, (int)d, (int)d, EPI_STORE, ep, s));
    for (int l = 0; l < m.depth; ++l) {
      const std::string p = "blocks." + std::to_string(l) + ".";
      ep.bias = WF(ctx, p + "xkv.b");
      ep.out = ctx->kv_text[l];
      ep.ldo = (int)(2 * d);
      CK(gemm(ctx, ctx->y, WT(ctx, p + "xkv.w"), (int)Mt, (int)(2 * d), (int)d, EPI_STORE, ep, s));
    }
    if (ctx->plan.cfg_split) {  // R33: each branch's text K/V rows, contiguous [L, 1, 2, d]
      for (int b = 0; b < 2; ++b) {
        if (ctx->kv_text_b[b].empty()) {
          ctx->kv_text_b[b].assign(m.depth, nullptr);
          for (auto &q : ctx->kv_text_b[b]) CK(dalloc(ctx, &q, (size_t)L * 2 * d * ctx->esz));
        }
        for (int l = 0; l < m.depth; ++l)
          CK(cudaMemcpy2DAsync(ctx->kv_text_b[b][l], (size_t)2 * d * ctx->esz,
                               (const char *)ctx->kv_text[l] + (size_t)b * 2 * d * ctx->esz,
                               (size_t)B * 2 * d * ctx->esz, (size_t)2 * d * ctx->esz, L,
                               cudaMemcpyDeviceToDevice, s));
      }
    }
  }
  return finish();
}
}  // namespace

extern "C" stadi_status stadi_num_steps(stadi_ctx *ctx, uint32_t *n) {
  ALIVE();
  if (!n) return ctx_fail(ctx, STADI_EINVAL, "NULL argument");
  if (!ctx->has_plan) return ctx_fail(ctx, STADI_ESTATE, "no plan installed");
  *n = (uint32_t)ctx->program.size();
  return STADI_OK;
}

// ---------------------------------------------------------------- exchange
namespace {

// Rows of group rank g in a slot (element offset, element count).
void seg_of(stadi_ctx *ctx, int g, int64_t *off, int64_t *cnt) {
  const Dims &m = ctx->dm;
  const int64_t per_tok = (int64_t)ctx->Bf * 2 * m.d;
  *off = (int64_t)ctx->plan.row_begin[g] / m.p * m.wp * per_tok;
  *cnt = (int64_t)ctx->plan.rows[g] / m.p * m.wp * per_tok;
}

// Publish the own rows of version `ver` at site l (after the QKV GEMM wrote them).
stadi_status publish(stadi_ctx *ctx, int li, int l, int ver, cudaStream_t s) {
  Rank &r = ctx->ranks[li];
  const int slot = l * 2 + (ver & 1);
  int64_t off, cnt;
  seg_of(ctx, r.g, &off, &cnt);
  const size_t bytes = cnt * ctx->esz;
  if (ctx->ipc_mode) {  // IPC: the QKV epilogue already stored the rows at the peers
    if (ctx->probe) return STADI_OK;
    ctx->exch_bytes += bytes * ctx->ipc->peers.size();
    return ipc_ready(ctx, l, ver, false, s);
  }
  if (!ctx->nccl) {  // local mode: copy into every other hosted rank's slot (same branch)
    for (auto &o : ctx->ranks) {
      if (o.g == r.g || o.branch != r.branch) continue;
      CK(cudaMemcpyAsync((char *)o.kv[slot] + off * ctx->esz, (char *)r.kv[slot] + off * ctx->esz,
                         bytes, cudaMemcpyDeviceToDevice, s));
      ctx->exch_bytes += bytes;
    }
    return STADI_OK;
  }
  // NCCL mode: in-place variable-size all-gather = one broadcast per included root
  CK(cudaEventRecord(ctx->ev_ready, s));
  CK(cudaStreamWaitEvent(ctx->comm, ctx->ev_ready, 0));
  const ncclDataType_t dt = ctx->dtype == STADI_DTYPE_BF16 ? ncclBfloat16 : ncclFloat32;
  CKN(nccl().GroupStart());
  int root = 0;
  for (uint32_t g = 0; g < ctx->plan.n_gpus; ++g) {
    if (!ctx->plan.tier[g]) continue;
    int64_t o2, c2;
    seg_of(ctx, (int)g, &o2, &c2);
    void *p = (char *)r.kv[slot] + o2 * ctx->esz;
    CKN(nccl().Broadcast(p, p, (size_t)c2, dt, root, ctx->sub_comm, ctx->comm));
    ++root;
  }
  CKN(nccl().GroupEnd());
  CK(cudaEventRecord(ctx->ev_done[slot], ctx->comm));
  ctx->ev_used[slot] = 1;
  ctx->exch_bytes += bytes;
  return STADI_OK;
}

// Make stream s wait until version `ver` of site l is complete (NCCL mode).
stadi_status wait_version(stadi_ctx *ctx, int l, int ver, cudaStream_t s) {
  if (!ctx->nccl || ver < 0) return STADI_OK;
  const int slot = l * 2 + (ver & 1);
  if (ctx->ev_used[slot])
    CK(timed(ctx, STADI_KCLASS_XWAIT, 0.0, 0.0, s,
             [&] { return cudaStreamWaitEvent(s, ctx->ev_done[slot], 0); }));
  return STADI_OK;
}


// One program step: patch-local forward of every part in layer lock-step,
// exchange at every attention site, then the Eq. 3 update of each band.
stadi_status run_phase(stadi_ctx *ctx, const std::vector<Part> &phase, cudaStream_t s) {
  if (ctx->dm.unet) return unet_run_phase(ctx, phase, s);
  const Dims &m = ctx->dm;
  const int64_t d = m.d;
  const int B = ctx->Bf;   // forward batch: 1 under the R33 CFG split, else the CFG batch
  const int BM = m.B;      // conditioning batch (mod / fmod rows per timestep)
  const int64_t mod_bs = (int64_t)m.depth * 6 * d;  // batch stride in mod
  const int ntok_full = m.hp * m.wp;
  for (const Part &P : phase) {  // x_res = patch embedding of the band (+ pos)
    Rank &r = ctx->ranks[P.li];
    CK(patch_embed(r.x_band, r.rows, m.lat_w, m.c_in, m.p, WF(ctx, "x_embed.w"),
                   WF(ctx, "x_embed.b"), ctx->pos_full + (int64_t)r.tok_begin * d, (int)d, B,
                   r.x_res, s));
  }
  for (int l = 0; l < m.depth; ++l) {
    const std::string pre = "blocks." + std::to_string(l) + ".";
    for (const Part &P : phase) {  // ---- LN/modulate + QKV (+ publish)
      Rank &r = ctx->ranks[P.li];
      const int M = r.n_tok * B;
      const float *mb = ctx->mod + ((int64_t)P.st.m * BM * m.depth + l) * 6 * d + r.branch * mod_bs;
      CK(lnmod(ctx, r.x_res, r.xmod, M, mb, mb + d, (int)mod_bs, 1, s));
      // own rows may only be overwritten once this rank's earlier sends of
      // the read version completed (NCCL mode)
      if (P.st.pub_ver != P.st.read_ver) ST(wait_version(ctx, l, P.st.read_ver, s));
      // IPC: the epilogue writes the publish version into the peers' slots; they
      // must be done reading that slot's previous version first
      const bool ipcx = ctx->ipc_mode && !ctx->probe && P.st.pub_ver >= 0;
      if (ipcx) ST(ipc_war_wait(ctx, l, P.st.pub_ver, false, s));
      EpiParams ep{};
      ep.bias = WF(ctx, pre + "qkv.b");
      ep.B = B;
      ep.q = r.q;
      ep.d = (int)d;
      ep.kv_a = r.kv[l * 2 + (P.st.read_ver & 1)];
      ep.kv_b = (P.st.pub_ver >= 0 && P.st.pub_ver != P.st.read_ver)
                    ? r.kv[l * 2 + (P.st.pub_ver & 1)]
                    : nullptr;
      ep.kv_row0 = (int64_t)r.tok_begin * B;
      if (ipcx) {
        ep.kv_peer = ipc_peer_slots(ctx, l, P.st.pub_ver & 1);
        ep.n_kv_peer = ep.kv_peer ? (int)ctx->ipc->peers.size() : 0;
      }
      CK(gemm(ctx, r.xmod, WT(ctx, pre + "qkv.w"), M, (int)(3 * d), (int)d, EPI_QKV, ep, s));
      if (P.st.pub_ver >= 0) ST(publish(ctx, P.li, l, P.st.pub_ver, s));
      if (P.st.pub_ver == P.st.read_ver) ST(wait_version(ctx, l, P.st.read_ver, s));  // fresh
    }
    for (const Part &P : phase) {  // ---- attention + rest of the block
      Rank &r = ctx->ranks[P.li];
      const int M = r.n_tok * B;
      const float *mb = ctx->mod + ((int64_t)P.st.m * BM * m.depth + l) * 6 * d + r.branch * mod_bs;
      const bool ipcr = ctx->ipc_mode && !ctx->probe;
      if (ipcr) ST(ipc_read_wait(ctx, l, P.st.read_ver, false, s));  // peers' rows of read_ver
      CK(attention(ctx, STADI_KCLASS_ATTN, r.q, r.kv[l * 2 + (P.st.read_ver & 1)], r.o, r.n_tok,
                    ntok_full, s));
      if (ipcr) ST(ipc_read_done(ctx, l, (uint32_t)P.idx + 1, false, s));
      EpiParams ep{};
      ep.B = B;
      ep.bias = WF(ctx, pre + "proj.b");
      ep.res = r.x_res;
      ep.ldr = (int)d;
      ep.gate = mb + 2 * d;
      ep.gate_bstride = (int)mod_bs;
      CK(gemm(ctx, r.o, WT(ctx, pre + "proj.w"), M, (int)d, (int)d, EPI_GATED_RES, ep, s));
      if (m.text) {  // cross-attention to the caption tokens (band-local)
        CK(lnmod(ctx, r.x_res, r.xmod, M, nullptr, nullptr, 0, 0, s));
        EpiParams eq{};
        eq.B = B;
        eq.bias = WF(ctx, pre + "xq.b");
        eq.out = r.q;
        eq.ldo = (int)d;
        CK(gemm(ctx, r.xmod, WT(ctx, pre + "xq.w"), M, (int)d, (int)d, EPI_STORE, eq, s));
        CK(attention(ctx, STADI_KCLASS_XATTN, r.q,
                     ctx->plan.cfg_split ? ctx->kv_text_b[r.branch][l] : ctx->kv_text[l], r.o,
                     r.n_tok, m.txt_len, s));
        EpiParams er{};
        er.B = B;
        er.bias = WF(ctx, pre + "xproj.b");
        er.res = r.x_res;
        er.ldr = (int)d;
        CK(gemm(ctx, r.o, WT(ctx, pre + "xproj.w"), M, (int)d, (int)d, EPI_RES, er, s));
      }
      CK(lnmod(ctx, r.x_res, r.xmod, M, mb + 3 * d, mb + 4 * d, (int)mod_bs, 1, s));
      EpiParams e1{};
      e1.B = B;
      e1.bias = WF(ctx, pre + "fc1.b");
      e1.out = r.h1;
      e1.ldo = (int)(4 * d);
      CK(gemm(ctx, r.xmod, WT(ctx, pre + "fc1.w"), M, (int)(4 * d), (int)d, EPI_GELU, e1, s));
      EpiParams e2{};
      e2.B = B;
      e2.bias = WF(ctx, pre + "fc2.b");
      e2.res = r.x_res;
      e2.ldr = (int)d;
      e2.gate = mb + 5 * d;
      e2.gate_bstride = (int)mod_bs;
      CK(gemm(ctx, r.h1, WT(ctx, pre + "fc2.w"), M, (int)d, (int)(4 * d), EPI_GATED_RES, e2, s));
    }
  }
  for (const Part &P : phase) {  // ---- final layer
    Rank &r = ctx->ranks[P.li];
    const int M = r.n_tok * B;
    const float *fb = ctx->fmod + (int64_t)P.st.m * BM * 2 * d + r.branch * 2 * d;
    CK(lnmod(ctx, r.x_res, r.xmod, M, fb, fb + d, (int)(2 * d), 1, s));
    EpiParams ef{};
    ef.B = B;
    ef.bias = ctx->final_b;
    // eps rows [n_tok, BM, fin_ld]; under the CFG split this rank fills its branch's
    ef.out = r.eps_raw + (ctx->plan.cfg_split ? r.branch * ctx->fin_ld : 0);
    ef.ldo = ctx->plan.cfg_split ? 2 * ctx->fin_ld : ctx->fin_ld;
    CK(gemm(ctx, r.xmod, ctx->final_w, M, ctx->fin_ld, (int)d, EPI_F32, ef, s));
  }
  const bool pair_ipc = ctx->plan.cfg_split && ctx->ipc_mode && !ctx->probe;
  if (ctx->plan.cfg_split && !ctx->probe) {  // R33: the pair swaps its eps rows
    for (const Part &P : phase) {
      Rank &r = ctx->ranks[P.li];
      if (pair_ipc) {
        ST(ipc_pair_push(ctx, m.depth, r.partner, (uint32_t)P.idx, r.eps_raw, r.n_tok,
                         ctx->fin_ld, r.branch, s));
        ST(ipc_pair_wait(ctx, m.depth, r.partner, (uint32_t)P.idx, s));
        continue;
      }
      for (auto &o : ctx->ranks)  // local mode: the partner is hosted here too
        if (o.g == r.partner) {
          const size_t pitch = (size_t)2 * ctx->fin_ld * 4;
          CK(cudaMemcpy2DAsync((char *)o.eps_raw + (size_t)r.branch * ctx->fin_ld * 4, pitch,
                               (const char *)r.eps_raw + (size_t)r.branch * ctx->fin_ld * 4,
                               pitch, (size_t)ctx->fin_ld * 4, r.n_tok,
                               cudaMemcpyDeviceToDevice, s));
          ctx->exch_bytes += (size_t)r.n_tok * ctx->fin_ld * 4;
        }
    }
  }
  for (const Part &P : phase) {  // ---- CFG + unpatchify + Eq. 3 on the band
    Rank &r = ctx->ranks[P.li];
    const int M = r.n_tok * BM;
    float A, Bc, Cz, c1, c2;
    sampler_coeffs(ctx, P.st.t, P.st.t_prev, &A, &Bc, &Cz);
    dpm2m_coeffs(ctx, r.sched, P.idx, &c1, &c2);
    const double sb = (double)r.rows * m.lat_w * m.c_in * 8 + (double)M * ctx->fin_ld * 4;
    CK(timed(ctx, STADI_KCLASS_SAMPLER, 0.0, sb, s, [&] {
      return sampler_update(r.x_band, r.eps_raw, r.rows, m.lat_w, m.c_in, m.p, m.c_out,
                            ctx->fin_ld, BM, m.guidance, A, Bc, Cz, ctx->ddpm_seed, ctx->seed_dev,
                            P.st.m, r.row_begin, s, r.hist, c1, c2);
    }));
    if (pair_ipc) ST(ipc_pair_done(ctx, m.depth, r.partner, (uint32_t)P.idx, s));
  }
  return STADI_OK;
}

}  // namespace

namespace {
// STADI_GRAPHS=0 disables the per-step CUDA graphs.
bool graphs_enabled(stadi_ctx *ctx) {
  static const int env = [] {
    const char *e = getenv("STADI_GRAPHS");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  // local mode, and IPC mode when the driver can capture its stream memory operations
  // (NCCL mode's cross-stream exchange events stay eager); not while per-launch kernel
  // timing is on (its events must see every launch)
  // Virtual GPUs (several contexts of one process) stay eager: a stream capture in one
  // thread can block behind another thread's synchronous pageable copy (which waits for
  // that rank's stream, which waits for this rank's flags): observed to deadlock.
  return env && !ctx->nccl && (!ctx->ipc_mode || ctx->ipc->graphs_ok) && !ctx->ktime &&
         !ctx->green_ctx;
}

// Program step i on stream s: replay its graph, capturing it on first use.
stadi_status exec_step(stadi_ctx *ctx, uint32_t i, cudaStream_t s) {
  if (!graphs_enabled(ctx)) return run_phase(ctx, ctx->program[i], s);
  if (ctx->graphs.size() != ctx->program.size()) ctx->graphs.assign(ctx->program.size(), {});
  auto &G = ctx->graphs[i];
  if (G.exec && G.emu_ctas != ctx->emu_ctas) {  // captured grids assume another free-SM count
    cudaGraphExecDestroy(G.exec);
    G.exec = nullptr;
  }
  static const bool dbg = getenv("STADI_DEBUG_GRAPHS") != nullptr;
  if (!G.exec) {
    // capture on the context's own stream (the caller's may be the legacy stream)
    if (dbg) fprintf(stderr, "[stadi r%d] step %u: sync\n", ctx->rank, i);
    CK(cudaEventRecord(ctx->ev_ready, s));  // host wait under the exchange watchdog
    ST(wait_event_watchdog(ctx, ctx->ev_ready));
    if (dbg) fprintf(stderr, "[stadi r%d] step %u: capture\n", ctx->rank, i);
    const unsigned long long l0 = g_launches;
    const uint64_t b0 = ctx->exch_bytes;
    CK(cudaStreamBeginCapture(ctx->gstream, cudaStreamCaptureModeThreadLocal));
    const stadi_status st = run_phase(ctx, ctx->program[i], ctx->gstream);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(ctx->gstream, &graph);
    if (st != STADI_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    CK(ec);
    if (dbg) fprintf(stderr, "[stadi r%d] step %u: instantiate\n", ctx->rank, i);
    const cudaError_t ei = cudaGraphInstantiate(&G.exec, graph, 0);
    cudaGraphDestroy(graph);
    CK(ei);
    G.launches = g_launches - l0;
    g_launches = l0;  // counted when the graph runs
    G.exch_bytes = ctx->exch_bytes - b0;
    ctx->exch_bytes = b0;
    G.emu_ctas = ctx->emu_ctas;
  }
  if (dbg) fprintf(stderr, "[stadi r%d] step %u: launch\n", ctx->rank, i);
  CK(cudaGraphLaunch(G.exec, s));
  ++ctx->graph_steps;
  g_launches += G.launches;
  ctx->exch_bytes += G.exch_bytes;
  return STADI_OK;
}
}  // namespace

extern "C" stadi_status stadi_denoise_step(stadi_ctx *ctx, uint32_t step, void *stream) {
  ALIVE();
  NvtxRange nv("stadi_denoise_step %u", step);
  ctx->last_stream = (cudaStream_t)stream;
  ctx->last_stream_set = true;
  if (!ctx->begun) return ctx_fail(ctx, STADI_ESTATE, "stadi_denoise_step before stadi_begin");
  if (step >= ctx->program.size()) return ctx_fail(ctx, STADI_EINVAL, "step out of range");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t w;
  CK(enter_stream(ctx, (cudaStream_t)stream, &w));
  ST(exec_step(ctx, step, w));
  CK(leave_stream(ctx, (cudaStream_t)stream));
  return STADI_OK;
}

namespace {
stadi_status gather_impl(stadi_ctx *ctx, float *out_full, void *stream) {
  if (!ctx->begun) return ctx_fail(ctx, STADI_ESTATE, "stadi_gather before stadi_begin");
  if (!out_full) return ctx_fail(ctx, STADI_EINVAL, "NULL argument");
  const Dims &m = ctx->dm;
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaSetDevice(ctx->device));
  const bool dev = is_device_ptr(out_full);
  const size_t row_elems = (size_t)m.lat_w * m.c_in;
  if (ctx->ipc_mode) return ipc_gather(ctx, out_full, dev, s);
  if (!ctx->nccl) {
    for (auto &r : ctx->ranks) {
      float *dst = out_full + (size_t)r.row_begin * row_elems;
      const size_t bytes = (size_t)r.rows * row_elems * 4;
      if (dev) CK(cudaMemcpyAsync(dst, r.x_band, bytes, cudaMemcpyDeviceToDevice, s));
      else CK(stage_d2h(ctx, dst, r.x_band, bytes, s));
    }
    return STADI_OK;
  }
  // NCCL: every rank (excluded ones too) receives every band (world communicator).
  // The exchange collectives run on the comm stream, possibly on the same
  // communicator: join it first so no two streams drive one communicator at once.
  CK(cudaEventRecord(ctx->ev_ready, ctx->comm));
  CK(cudaStreamWaitEvent(s, ctx->ev_ready, 0));
  float *full = nullptr;
  CK(cudaMallocAsync(&full, (size_t)m.lat_h * row_elems * 4, s));
  if (!ctx->ranks.empty())
    CK(cudaMemcpyAsync(full + (size_t)ctx->ranks[0].row_begin * row_elems, ctx->ranks[0].x_band,
                       (size_t)ctx->ranks[0].rows * row_elems * 4, cudaMemcpyDeviceToDevice, s));
  CKN(nccl().GroupStart());
  for (uint32_t g = 0; g < ctx->plan.n_gpus; ++g) {
    if (!ctx->plan.rows[g]) continue;
    float *p = full + (size_t)ctx->plan.row_begin[g] * row_elems;
    CKN(nccl().Broadcast(p, p, (size_t)ctx->plan.rows[g] * row_elems, ncclFloat32, (int)g,
                         ctx->world_comm, s));
  }
  CKN(nccl().GroupEnd());
  if (dev)
    CK(cudaMemcpyAsync(out_full, full, (size_t)m.lat_h * row_elems * 4, cudaMemcpyDeviceToDevice,
                       s));
  else
    CK(stage_d2h(ctx, out_full, full, (size_t)m.lat_h * row_elems * 4, s));
  CK(cudaFreeAsync(full, s));
  return STADI_OK;
}
}  // namespace

extern "C" stadi_status stadi_run(stadi_ctx *ctx, const stadi_plan_t *plan, const float *noise_full,
                                  const stadi_cond *cond, float *out_full, stadi_run_stats *stats,
                                  void *stream) {
  ALIVE();
  NvtxRange nv("stadi_run");
  if (!plan || !noise_full || !cond || !out_full)
    return ctx_fail(ctx, STADI_EINVAL, "NULL argument");
  CK(cudaSetDevice(ctx->device));
  DBG("run: start");
  if (!ctx->has_plan || std::memcmp(plan, &ctx->plan, sizeof(stadi_plan_t)) != 0)
    ST(stadi_set_plan(ctx, plan));
  DBG("run: plan installed");
  cudaStream_t s;
  CK(enter_stream(ctx, (cudaStream_t)stream, &s));
  ctx->last_stream = s;
  ctx->last_stream_set = true;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const unsigned long long l0 = g_launches;
  CK(collect_timing(ctx));  // (no-op unless timing) so the exchange-wait delta is this request's
  ctx->graph_steps = 0;
  const double w0 = ctx->kt[STADI_KCLASS_XWAIT].ms;
  CK(cudaEventRecord(e0, s));
  ST(begin_impl(ctx, noise_full, cond, s));
  DBG("run: begun");
  for (uint32_t i = 0; i < ctx->program.size(); ++i) ST(exec_step(ctx, i, s));
  DBG("run: steps enqueued");
  ST(gather_impl(ctx, out_full, s));
  DBG("run: gather enqueued");
  CK(cudaEventRecord(e1, s));
  CK(leave_stream(ctx, (cudaStream_t)stream));
  ST(wait_event_watchdog(ctx, e1));
  DBG("run: done");
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CK(collect_timing(ctx));
  if (stats) {
    stats->ms_total = ms;
    stats->ms_exchange_wait = ctx->kt[STADI_KCLASS_XWAIT].ms - w0;
    stats->exchange_bytes = ctx->exch_bytes;
    stats->kernel_launches = (uint32_t)(g_launches - l0);
    stats->steps_run = (uint32_t)ctx->program.size();
    stats->graph_steps = ctx->graph_steps;
  }
  return STADI_OK;
}

// ---------------------------------------------------------------- profiling (a1)
namespace {
stadi_status profile_impl(stadi_ctx *ctx, uint32_t n_steps, const uint32_t *units, double *ms_out,
                          uint64_t *speed_out);
}
extern "C" stadi_status stadi_profile_warmup(stadi_ctx *ctx, uint32_t n_steps, double *ms_out,
                                             uint64_t *speed_out) {
  ALIVE();
  NvtxRange nv("stadi_profile_warmup");
  if (!ms_out || !speed_out || n_steps == 0) return ctx_fail(ctx, STADI_EINVAL, "bad argument");
  return profile_impl(ctx, n_steps, nullptr, ms_out, speed_out);
}
extern "C" stadi_status stadi_profile_band(stadi_ctx *ctx, uint32_t n_steps, const uint32_t *units,
                                           double *ms_out) {
  ALIVE();
  NvtxRange nv("stadi_profile_band");
  if (!ms_out || !units || n_steps == 0) return ctx_fail(ctx, STADI_EINVAL, "bad argument");
  std::vector<uint64_t> sp(ctx->G);
  return profile_impl(ctx, n_steps, units, ms_out, sp.data());
}

namespace {
stadi_status profile_impl(stadi_ctx *ctx, uint32_t n_steps, const uint32_t *units, double *ms_out,
                          uint64_t *speed_out) {
  if (!ctx->weights_loaded) return ctx_fail(ctx, STADI_ESTATE, "weights not loaded");
  const Dims &m = ctx->dm;
  CK(cudaSetDevice(ctx->device));
  // uniform probe plan over the whole group (Eq. 5 with equal speeds)
  std::vector<uint64_t> ones(ctx->G, 1);
  stadi_plan_params pp{};
  pp.n_gpus = ctx->G;
  pp.speed = ones.data();
  pp.m_base = 10;
  pp.m_warmup = 10;
  pp.a_num = 3; pp.a_den = 4; pp.b_num = 1; pp.b_den = 4;
  pp.rows_per_unit = m.unet ? (1u << (m.levels() - 1)) : (uint32_t)m.p;
  pp.p_total = m.lat_h / pp.rows_per_unit;
  pp.flags = STADI_NO_TA | STADI_NO_SA;
  if (units) {  // stadi_profile_band: the caller's band sizes (forced units, R6 units)
    pp.flags |= STADI_FORCE_UNITS;
    pp.forced_units = units;
  }
  if ((int)pp.p_total < ctx->G) return ctx_fail(ctx, STADI_EINVAL, "latent too small for group");
  stadi_plan_t probe;
  if (stadi_plan(&pp, &probe) != STADI_OK)
    return ctx_fail(ctx, STADI_EINVAL, "probe plan: %s", tls_error().c_str());
  ST(stadi_set_plan(ctx, &probe));
  std::vector<float> zeros((size_t)m.lat_h * m.lat_w * m.c_in, 0.f);
  std::vector<int32_t> labels(m.B, 0);
  std::vector<float> text, pooled;
  stadi_cond cond{labels.data(), nullptr, nullptr, nullptr};
  if (m.text) {
    text.assign((size_t)m.B * m.txt_len * m.txt_dim, 0.f);
    cond.text = text.data();
  }
  if (m.add_embed) {
    pooled.assign((size_t)m.B * m.pooled_dim, 0.f);
    cond.pooled = pooled.data();
  }
  cudaStream_t s = ctx->green_ctx ? ctx->wstream : nullptr;
  ST(begin_impl(ctx, zeros.data(), &cond, s));
  std::vector<double> ms_local(ctx->ranks.size(), 0.0);
  ctx->probe = true;  // compute-only probe steps: no exchange waits / signals
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (size_t li = 0; li < ctx->ranks.size(); ++li) {
    std::vector<double> v;
    // compute-only probe step: reads version 0, publishes nothing (no waits)
    Part P{(int)li, stadi_step_t{0, 901, 801, STADI_STEP_UNIFORM, 0, STADI_VER_NONE}};
    for (uint32_t it = 0; it <= n_steps; ++it) {
      CK(cudaEventRecord(e0, s));
      ST(run_phase(ctx, {P}, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (it > 0) v.push_back(ms);  // first one is a warm-up
    }
    std::sort(v.begin(), v.end());
    ms_local[li] = v[v.size() / 2];
  }
  ctx->probe = false;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  std::vector<double> all(ctx->G, 0.0);
  if (ctx->ipc_mode) {
    ST(ipc_allgather_f64(ctx, ms_local.empty() ? 0.0 : ms_local[0], all));
  } else if (!ctx->nccl) {
    for (size_t li = 0; li < ctx->ranks.size(); ++li) all[ctx->ranks[li].g] = ms_local[li];
  } else {
    double *dsend = nullptr, *drecv = nullptr;
    CK(pmalloc(ctx, &dsend, 8));
    CK(pmalloc(ctx, &drecv, 8 * ctx->G));
    CK(cudaStreamSynchronize(ctx->astream));
    CK(cudaMemcpy(dsend, ms_local.data(), 8, cudaMemcpyHostToDevice));
    CKN(nccl().AllGather(dsend, drecv, 1, ncclFloat64, ctx->world_comm, s));
    CK(cudaMemcpy(all.data(), drecv, 8 * ctx->G, cudaMemcpyDeviceToHost));
    pfree(ctx, dsend);
    pfree(ctx, drecv);
  }
  double mn = all[0];
  for (double x : all) mn = std::min(mn, x);
  for (int g = 0; g < ctx->G; ++g) {
    ms_out[g] = all[g];
    speed_out[g] = (uint64_t)std::llround(1048576.0 * mn / all[g]);
    if (!speed_out[g]) speed_out[g] = 1;
  }
  free_plan_buffers(ctx);
  return STADI_OK;
}
}  // namespace

// ---------------------------------------------------------------- emulator (a9)
extern "C" stadi_status stadi_emulator_start(stadi_ctx *ctx, uint32_t pct) {
  ALIVE();
  if (pct > 95) return ctx_fail(ctx, STADI_EINVAL, "occupancy must be <= 95%%");
  if (ctx->emu_ctas) return ctx_fail(ctx, STADI_ESTATE, "emulator already running");
  if (pct == 0) return STADI_OK;
  CK(cudaSetDevice(ctx->device));
  const int n = emulator_ctas((int)pct, ctx->num_sms);
  // every kernel the context may launch while the emulator is resident must be
  // loaded now (lazy loading may need a context sync: it would wait for the
  // emulator forever); the SIMT kernels are loaded by this context's earlier work
  // or by the bench's profiling pass, the tcgen05 variants depend on the free SMs
  if (ctx->dtype == STADI_DTYPE_BF16) {
    CK(tc_gemm_preload());
    CK(tc_attention_preload());
  }
  CK(cudaMemsetAsync(ctx->emu_flag_dev, 0, 4, ctx->emu_stream));
  CK(emulator_launch(n, ctx->emu_flag_dev, ctx->emu_stream));
  ctx->emu_ctas = n;
  return STADI_OK;
}

extern "C" stadi_status stadi_emulator_stop(stadi_ctx *ctx) {
  ALIVE();
  if (!ctx->emu_ctas) return STADI_OK;
  CK(cudaMemsetAsync(ctx->emu_flag_dev, 1, 4, ctx->emu_ctl));  // nonzero: stop
  CK(cudaStreamSynchronize(ctx->emu_stream));
  ctx->emu_ctas = 0;
  return STADI_OK;
}

// ---------------------------------------------------------------- kernel timing (d)
extern "C" stadi_status stadi_kernel_timing(stadi_ctx *ctx, int32_t enable) {
  ALIVE();
  CK(cudaSetDevice(ctx->device));
  CK(quiesce(ctx));
  for (auto &k : ctx->kt) {
    k.used = 0;
    k.launches = 0;
    k.ms = k.flops = k.bytes = 0;
  }
  ctx->ktime = enable != 0;
  return STADI_OK;
}

extern "C" stadi_status stadi_kernel_stats(stadi_ctx *ctx, int32_t kclass, uint64_t *launches,
                                           double *ms, double *flops, double *bytes) {
  ALIVE();
  if (kclass < 0 || kclass >= STADI_KCLASS_COUNT)
    return ctx_fail(ctx, STADI_EINVAL, "unknown kernel class %d", kclass);
  CK(cudaSetDevice(ctx->device));
  CK(quiesce(ctx));
  CK(collect_timing(ctx));
  const auto &k = ctx->kt[kclass];
  if (launches) *launches = k.launches;
  if (ms) *ms = k.ms;
  if (flops) *flops = k.flops;
  if (bytes) *bytes = k.bytes;
  return STADI_OK;
}
