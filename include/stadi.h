/*
 * stadi.h — C ABI of the B200-native STADI elastic patch-parallel denoiser.
 *
 * STADI = Spatio-Temporal Adaptive Diffusion Inference, arXiv 2509.04719
 * (/root/reference/PAPER.md).  The boundary follows the paper's statement of
 * the problem: inputs are an initial noise x_{t_0}, a model eps_theta, the
 * effective speeds {v_i}, M_base and M_warmup (Alg. 1 inputs, L108-L112);
 * outputs are the final image x_{t_M} (L113) and the assignment (M_i, P_i)
 * per GPU (§III-B).
 *
 * The four north-star calls:
 *   stadi_profile_warmup  per-GPU speed v_i from timed warm-up forwards
 *                         (L179 "effective speed", L284-L286 "derived directly
 *                         from historical inference time profiles")
 *   stadi_plan            Eq. 4 step allocation + Eq. 5 patch sizing
 *                         (L179-L198, Alg. 1 lines 1-6)
 *   stadi_denoise_step    one patch-parallel model forward + Eq. 3 sampler
 *                         update on this GPU's patch (Alg. 1 lines 9-24)
 *   stadi_run             a full request (Alg. 1 end to end, line 25)
 *
 * Conventions (all calls):
 *   - Every call returns stadi_status; nothing throws or aborts.
 *     STADI_EINVAL: bad arguments (no state change).  STADI_ECUDA /
 *     STADI_ENCCL: a CUDA / NCCL error; the context is poisoned and only
 *     stadi_destroy is valid afterwards (later calls return STADI_ESTATE).
 *     stadi_last_error(ctx) gives a human-readable message (ctx may be NULL:
 *     thread-local message of the last context-less call).
 *   - Ownership: the caller owns every pointer it passes; the library copies
 *     what it keeps (plans, conditioning, weights).  Device pointers must be
 *     on the context's device and stay valid until the enqueued work ends.
 *     The context owns its weights, activations, exchange buffers, streams,
 *     events and communicators.
 *   - Streams are passed as `void *` holding a cudaStream_t (NULL = legacy
 *     default stream).  denoise_step / gather are stream-ordered; stadi_run
 *     synchronises before returning.
 *   - "COLLECTIVE" calls must be made by every rank of the group in the same
 *     order with identical plans (the plan is a pure function of speed[]).
 *   - One host thread per context.
 *
 * Layouts: latents are NHWC float32, [H, W, C] row-major for the full image,
 * a rank's patch p_i is the contiguous row band [row_begin_i, row_begin_i +
 * rows_i) (rank order, top to bottom).
 */
#ifndef STADI_H_
#define STADI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STADI_ABI_VERSION 3u
#define STADI_MAX_GPUS 64

typedef enum {
  STADI_OK = 0,
  STADI_EINVAL = 1,
  STADI_ENOMEM = 2,
  STADI_ECUDA = 3,
  STADI_ENCCL = 4,
  STADI_ESTATE = 5,        /* poisoned context or wrong call order          */
  STADI_EUNSUPPORTED = 6
} stadi_status;

typedef struct stadi_ctx stadi_ctx;

uint32_t stadi_abi_version(void);
const char *stadi_status_str(stadi_status s);
/* Last error message of ctx (or of this thread when ctx == NULL).  Valid until
 * the next call on the same ctx / thread. */
const char *stadi_last_error(const stadi_ctx *ctx);

/* ======================================================================
 * Planner — pure host, integer only, deterministic, re-entrant, no CUDA.
 * ====================================================================== */
enum {
  STADI_NO_TA = 1u,           /* disable temporal adaptation (every GPU tier 1) */
  STADI_NO_SA = 2u,           /* disable spatial adaptation (uniform units)     */
  STADI_SIZER_INTERVAL = 4u,  /* Eq. 5 with per-round step counts (R7 variant)  */
  STADI_FORCE_UNITS = 8u,     /* use forced_units (Table II / Fig. 9 splits)    */
  STADI_SIZER_AFFINE = 16u,   /* Eq. 5 replaced by the affine step-cost model
                                 alpha_i + beta_i P (R30, L333 fixed overhead)  */
  STADI_CFG_SPLIT = 32u       /* R33: CFG batch split -- GPUs paired by speed, each
                                 member computes one CFG branch of the pair's band
                                 (B = 1), Eq. 4/5 plan the pairs (speed = min of the
                                 pair); not with FORCE_UNITS / SIZER_AFFINE         */
};

typedef struct {
  uint32_t n_gpus;             /* N, 1..STADI_MAX_GPUS                           */
  const uint64_t *speed;       /* [N] effective speeds v_i > 0, any common scale */
  uint32_t m_base, m_warmup;   /* 1 <= M_warmup <= M_base (L284: 100 / 4)        */
  uint32_t a_num, a_den;       /* a = a_num/a_den, 0 < b < a < 1 (L284: 3/4)     */
  uint32_t b_num, b_den;       /* b (L284: 1/4)                                  */
  uint32_t p_total;            /* P_total units (L284: 32); >= #included GPUs    */
  uint32_t rows_per_unit;      /* latent rows per unit (R6)                      */
  uint32_t flags;              /* STADI_NO_TA | STADI_NO_SA | ...                */
  const uint32_t *forced_units;/* [N] with STADI_FORCE_UNITS, else ignored       */
  const uint64_t *alpha;       /* [N] with STADI_SIZER_AFFINE: fixed per-step cost
                                  of GPU i (any integer time unit), else ignored */
  const uint64_t *beta;        /* [N] with STADI_SIZER_AFFINE: per-step cost of one
                                  unit on GPU i (> 0 for included GPUs)          */
} stadi_plan_params;

typedef struct {
  uint32_t n_gpus, m_base, m_warmup, p_total, rows_per_unit;
  uint8_t tier[STADI_MAX_GPUS];        /* Eq. 4: 1 = M_base, 2 = (M_base+M_warmup)/2,
                                          0 = excluded (v_i <= b v_max)          */
  uint32_t steps[STADI_MAX_GPUS];      /* M_i (0 when excluded)                   */
  uint32_t units[STADI_MAX_GPUS];      /* P_i in units (Eq. 5, D'Hondt, R5)       */
  uint32_t row_begin[STADI_MAX_GPUS];  /* first latent row of GPU i's band        */
  uint32_t rows[STADI_MAX_GPUS];       /* latent rows of GPU i's band             */
  uint32_t sync_period;                /* lcm of post-warmup DDIM strides = the
                                          tier-2 stride n: 1 (nobody slow), 2 (K =
                                          M_base - M_warmup even), else the smallest
                                          prime factor of K (R32)                 */
  uint32_t n_exchange_rounds;          /* M_warmup + (M_base-M_warmup)/sync_period */
  uint64_t makespan_num, makespan_den; /* max_i M_i P_i / v_i, reduced fraction
                                          (SIZER_AFFINE: max_i M_i (alpha_i +
                                          beta_i P_i), den 1)                     */
  uint32_t cfg_split;                  /* 1: STADI_CFG_SPLIT plan (R33)           */
  uint8_t branch[STADI_MAX_GPUS];      /* CFG branch of GPU i (0 uncond, 1 cond)  */
  int8_t partner[STADI_MAX_GPUS];      /* the other member of GPU i's pair, or -1 */
} stadi_plan_t;

/* Eq. 4 (L179-L185) then Eq. 5 (L187-L198), as in Alg. 1 lines 1-6.
 * Thresholds compared exactly in 128-bit integers (R2: v_i <= b v_max is
 * excluded, tier 1 needs a v_max < v_i).  Eq. 5 is integerised with the
 * D'Hondt divisor method (R5): one unit per included GPU, then each further
 * unit to argmin (P_i + 1) M_i / v_i, ties to the lowest rank.  With
 * STADI_SIZER_AFFINE (R30, L333: "the single-step delay no longer maintains a
 * linear relationship with the patch size due to some fixed overhead") each
 * further unit goes to argmin M_i (alpha_i + beta_i (P_i + 1)) instead, which
 * minimises max_i M_i (alpha_i + beta_i P_i); Eq. 4 still uses speed.
 * Tier 2 runs M_warmup + K/n steps, K = M_base - M_warmup, stride n = 2 for even K
 * ((M_base + M_warmup)/2 as printed in Eq. 4), else the smallest prime factor of K
 * (R32, keeps Thm 2's aligned grids).
 * EINVAL: N out of range, a zero speed, not 0<b<a<1, M_warmup out of range,
 * P_total < #included, bad
 * forced units, SIZER_AFFINE without alpha / beta or with beta_i == 0 on an
 * included GPU. */
stadi_status stadi_plan(const stadi_plan_params *in, stadi_plan_t *out);

enum {
  STADI_STEP_WARMUP = 0,     /* Alg. 1: synchronous (fresh) exchange   */
  STADI_STEP_UNIFORM = 1,    /* no slow GPU: every step exchanges (R13)          */
  STADI_STEP_FAST_EVEN = 2,  /* L136-L140: async buffer update + all-gather      */
  STADI_STEP_FAST_ODD = 3,   /* L142-L146: no buffer update, reads newest (R10)  */
  STADI_STEP_SLOW = 4        /* L148-L152: stride-2 step, async buffer update    */
};
#define STADI_T_FINAL (-1)   /* t_prev of the last step: alpha_bar_0 (R18)       */
#define STADI_VER_NONE (-1)  /* pub_ver of a step that publishes nothing         */

typedef struct {
  int32_t m;          /* fast-grid index                                        */
  int32_t t, t_prev;  /* DDIM timesteps (leading spacing, offset 1, R18)         */
  int32_t kind;       /* STADI_STEP_*                                            */
  int32_t read_ver;   /* exchange version read at every site (== pub_ver: fresh) */
  int32_t pub_ver;    /* version published, or STADI_VER_NONE                    */
} stadi_step_t;

/* Step table of one rank (Alg. 1, Thm 2 grid alignment L234-L238).
 * Writes min(cap, n) entries to buf and the full count to *n_out (buf may be
 * NULL with cap 0 to query the count). */
stadi_status stadi_schedule(const stadi_plan_t *plan, uint32_t rank,
                            stadi_step_t *buf, uint32_t cap, uint32_t *n_out);

/* ======================================================================
 * Model description and weights
 * ====================================================================== */
enum {
  STADI_PRESET_TINY_DIT = 0,   /* C1: d 64, 4 heads, depth 2, 16x16x4 latent    */
  STADI_PRESET_DIT_XL2 = 1,    /* C2: DiT-XL/2 shapes, 32x32x4 latent, CFG 4.0  */
  STADI_PRESET_PIXART_ALPHA = 2,/* C5: PixArt-alpha shapes, 256x256x4, CFG 4.5  */
  STADI_PRESET_SD15 = 3,       /* C3: SD-1.5 U-Net shapes, 64x64x4, CFG 7.5      */
  STADI_PRESET_SDXL = 4,       /* C4: SDXL U-Net shapes, 128x128x4, CFG 5.0      */
  STADI_PRESET_TINY_UNET = 5   /* 2-level U-Net for fast parity tests            */
};
enum { STADI_DTYPE_BF16 = 0, STADI_DTYPE_FP32_DEBUG = 1 };
/* DDIM: Eq. 3.  DDPM: Eq. 2 (L62) realised as the eta = 1
 * step of ref. [28] (R19): x' = alpha' x0_hat + sqrt(1 - abar' - s^2) eps + s z_m,
 * s = sqrt((1 - abar')/(1 - abar)) sqrt(1 - abar/abar'), z_m drawn in the
 * sampler kernel from the counter-based generator keyed by stadi_cond.ddpm_seed. */
/* DPM2M: R34, the multistep DPM-Solver-2 of Lu et al. (L66 "higher-order solvers",
 * refs [31], [32]) in noise-prediction form: Eq. 3 with eps replaced by
 * eps + (eps - eps_prev) / (2 r), r = h_prev / h, eps_prev the band's previous own
 * step (first step: Eq. 3). */
enum { STADI_SAMPLER_DDIM = 0, STADI_SAMPLER_DDPM = 1, STADI_SAMPLER_DPM2M = 2 };

typedef struct {
  int32_t preset;          /* STADI_PRESET_*                                     */
  int32_t dtype;           /* BF16: tcgen05 bf16 GEMM/attention, fp32 accumulate,
                              fp32 residual + latent; FP32_DEBUG: SIMT fp32 (no
                              TF32) kernels for the <=1e-4 parity build         */
  int32_t sampler;         /* STADI_SAMPLER_DDIM | _DDPM | _DPM2M (EINVAL else)   */
  int32_t depth;           /* 0 = preset depth; >0: DiT blocks, or the cap on every
                              U-Net transformer depth (reduced parity variants)  */
  int32_t latent_h, latent_w; /* 0 = preset resolution                           */
} stadi_model_desc;

/* Weight manifest: tensors in load order (same order as synth/configs.py
 * manifest()).  Linear weights are [out, in] row-major float32. */
stadi_status stadi_weight_count(const stadi_model_desc *desc, uint32_t *n_tensors);
stadi_status stadi_weight_info(const stadi_model_desc *desc, uint32_t index,
                               char *name_buf, uint32_t name_cap, uint64_t *numel);

/* ======================================================================
 * Runtime — one context per process; a context hosts one rank (world > 1,
 * NCCL over NVLink) or n_local ranks on one device (world == 1; exchange by
 * device copies — used to run the multi-rank protocol on a single GPU).
 * ====================================================================== */
/* Transport of the exchange when world > 1 (one rank per process):
 *  NCCL: grouped ncclBroadcast / ncclAllGather on a high-priority side stream
 *        (the variable-size all-gather of L288); one GPU per process.
 *  IPC:  one-sided, CUDA IPC between the processes of ONE node (any GPUs with
 *        peer access, or several processes sharing one GPU): the QKV GEMM
 *        epilogue stores its K/V rows straight into the peers' slots (the
 *        all-gather fused into the producer), halo rows go to the two
 *        neighbour ranks only, GroupNorm partials to all, and completion is
 *        signalled by stream memory operations on flags in the receiver's
 *        memory (no SM spins, no host round trips).  nccl_id then carries a
 *        128-byte session id (stadi_ipc_session_id) that namespaces the
 *        node-local control files (/dev/shm) used to swap IPC handles. */
enum { STADI_TRANSPORT_NCCL = 0, STADI_TRANSPORT_IPC = 1 };

typedef struct {
  int32_t rank, world;       /* process rank / number of processes               */
  int32_t device;            /* CUDA device ordinal                              */
  int32_t n_local;           /* ranks hosted by this ctx (>1 only if world == 1) */
  const uint8_t *nccl_id;    /* 128 bytes from rank 0 when world > 1: the
                                ncclUniqueId (NCCL) or the session id (IPC)      */
  int32_t transport;         /* STADI_TRANSPORT_* (world > 1)                    */
  int32_t vgpu_sms;          /* 0: the whole device.  > 0 (multiple of 8): a
                                VIRTUAL GPU -- every kernel of the context runs in
                                green-context SM partition number `rank` of this
                                many SMs (disjoint per rank), so several contexts
                                of one process, one per host thread, compute a
                                multi-rank request concurrently on one device
                                (IPC transport between them; HBM / L2 shared).
                                A NULL stream argument then means the context's
                                own stream (the legacy stream is not joined: it
                                is shared by all threads of the process).
                                EUNSUPPORTED if the partition does not fit       */
} stadi_dist_desc;

typedef struct {
  const int32_t *labels;     /* [B] class labels (class presets; B=2: null first)  */
  const float *text;         /* [B, L_txt, D_txt] fp32, host or device (text presets;
                                B=2: the null caption first)                        */
  const float *pooled;       /* [B, 1280] fp32 pooled text embedding (SDXL), host or
                                device; NULL for other presets                      */
  const float *time_ids;     /* [B, 6] host fp32 SDXL micro-conditioning, or NULL =
                                the preset's (1024, 1024, 0, 0, 1024, 1024)         */
  uint64_t ddpm_seed;        /* STADI_SAMPLER_DDPM: key of the request's noise draws
                                z_m (R19: Philox4x64-10, key (ddpm_seed, m), counter
                                = full-image element index / 4, Box-Muller); ignored
                                by DDIM                                              */
} stadi_cond;

typedef struct {
  double ms_total;           /* device time of the request on this process       */
  double ms_exchange_wait;   /* device time the compute stream spent blocked on
                                exchange completion (NCCL events / IPC flags);
                                measured only while kernel timing is enabled
                                (stadi_kernel_timing), else 0                   */
  uint64_t exchange_bytes;   /* bytes this process sent in exchange rounds       */
  uint32_t kernel_launches;  /* kernels this process launched for the request    */
  uint32_t steps_run;        /* program steps executed                           */
  uint32_t graph_steps;      /* of which replayed from per-step CUDA graphs      */
} stadi_run_stats;

stadi_status stadi_create(const stadi_model_desc *model, const stadi_dist_desc *dist,
                          stadi_ctx **out);
void stadi_destroy(stadi_ctx *ctx);

/* Copy the weights (host float32, manifest order) to the device, converting
 * GEMM operands to the context dtype.  EINVAL on count / numel mismatch. */
stadi_status stadi_load_weights(stadi_ctx *ctx, uint32_t n_tensors,
                                const float *const *host_tensors, const uint64_t *numels);

/* COLLECTIVE.  Times n_steps compute-only forwards on a uniform band (no
 * exchange waits), takes the median ms per step ms_i, all-gathers it and
 * returns v_i = round(2^20 min_j ms_j / ms_i) (R1).  ms_out / speed_out: [G]
 * where G = world * n_local. */
stadi_status stadi_profile_warmup(stadi_ctx *ctx, uint32_t n_steps, double *ms_out,
                                  uint64_t *speed_out);

/* COLLECTIVE.  As stadi_profile_warmup, with the probe band of group rank g forced
 * to units[g] planner units (sum = the latent's units; every entry >= 1): two
 * calls with different sizes give each GPU's per-step cost alpha_g + beta_g P, the
 * input of STADI_SIZER_AFFINE (R30; L333 "fixed overhead").  ms_out: [G]. */
stadi_status stadi_profile_band(stadi_ctx *ctx, uint32_t n_steps, const uint32_t *units,
                                double *ms_out);

/* COLLECTIVE.  Install a plan (n_gpus == G, p_total * rows_per_unit == latent
 * height).  Allocates bands and exchange slots. */
stadi_status stadi_set_plan(stadi_ctx *ctx, const stadi_plan_t *plan);

/* Start a request: take this context's rows of the full noise [H, W, C_in]
 * (host or device pointer) and the conditioning; precompute per-timestep
 * modulation and text K/V.  Stream-ordered on `stream`.  COLLECTIVE with the
 * IPC transport (resets the exchange flags behind a device-side barrier). */
stadi_status stadi_begin(stadi_ctx *ctx, const float *noise_full, const stadi_cond *cond,
                         void *stream);
/* Number of program steps of the installed plan (local mode: steps grouped by
 * fast-grid index m across the hosted ranks; NCCL mode: this rank's steps). */
stadi_status stadi_num_steps(stadi_ctx *ctx, uint32_t *n);
/* COLLECTIVE.  Program step i: patch-local forward with stale exchange + Eq. 3
 * update of the hosted bands (Alg. 1 lines 9-24). */
stadi_status stadi_denoise_step(stadi_ctx *ctx, uint32_t step, void *stream);
/* COLLECTIVE.  Final synchronous all-gather of the bands into out_full [H, W, C]
 * fp32 (host or device pointer). */
stadi_status stadi_gather(stadi_ctx *ctx, float *out_full, void *stream);
/* COLLECTIVE.  set_plan (if changed) + begin + every step + gather; synchronises.
 * noise_full / out_full may be host or device pointers. */
stadi_status stadi_run(stadi_ctx *ctx, const stadi_plan_t *plan, const float *noise_full,
                       const stadi_cond *cond, float *out_full, stadi_run_stats *stats,
                       void *stream);

/* Occupancy emulator (R24): take ceil(pct * SMs / 100) SMs,
 * rounded up to an even count (whole TPCs, so the free SMs still form the CTA
 * pairs of the cta_group::2 GEMMs), with a resident kernel whose CTAs hold all of
 * an SM's shared memory, threads and registers and sleep until stopped (hard
 * self-timeout 900 s).  The context's persistent GEMM grids shrink to the free
 * SMs.  ESTATE if already running; EINVAL for pct > 95. */
stadi_status stadi_emulator_start(stadi_ctx *ctx, uint32_t occupancy_pct);
stadi_status stadi_emulator_stop(stadi_ctx *ctx);

/* Per-class kernel timing (measurement).  When enabled, every
 * launch of a timed class is bracketed by two CUDA events recorded on the
 * stream the kernel is launched on; stadi_kernel_stats synchronises the
 * device, folds the events in and returns, for the class, the number of
 * launches, their summed device time in ms and their summed ALGORITHMIC work
 * (flops: 2 per multiply-add of the layer's definition, attention = QK^T + PV;
 * bytes: the kernel's compulsory HBM reads + writes).  Enabling (or
 * re-enabling) resets the totals.  EINVAL for an unknown class. */
enum {
  STADI_KCLASS_GEMM = 0,     /* every tcgen05 / SIMT linear layer              */
  STADI_KCLASS_ATTN = 1,     /* self-attention, own Q x full (stale) K/V       */
  STADI_KCLASS_XATTN = 2,    /* cross-attention to the text tokens             */
  STADI_KCLASS_NORM = 3,     /* LayerNorm + adaLN modulate                     */
  STADI_KCLASS_SAMPLER = 4,  /* CFG + unpatchify + Eq. 3 update                */
  STADI_KCLASS_XWAIT = 5,    /* exchange waits (no kernel: the time the stream
                                is blocked on a peer's version; flops = bytes = 0) */
  STADI_KCLASS_COUNT = 6
};
stadi_status stadi_kernel_timing(stadi_ctx *ctx, int32_t enable);
stadi_status stadi_kernel_stats(stadi_ctx *ctx, int32_t kclass, uint64_t *launches, double *ms,
                                double *flops, double *bytes);

/* ncclGetUniqueId through the library's NCCL (dlopen'ed; ENCCL if absent). */
stadi_status stadi_nccl_unique_id(uint8_t out[128]);
/* A fresh random session id for the IPC transport (rank 0 calls it and
 * broadcasts the bytes, like an ncclUniqueId). */
stadi_status stadi_ipc_session_id(uint8_t out[128]);

#ifdef __cplusplus
}
#endif
#endif /* STADI_H_ */
