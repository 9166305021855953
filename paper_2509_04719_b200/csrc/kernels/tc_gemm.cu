// tcgen05 + TMA bf16 GEMM for sm_100a:  out = epilogue(A[M,K] . W[N,K]^T).
//
// Every linear layer of the patch-local DiT block (QKV, out-proj, MLP, final
// layer, adaLN / caption / cross-K/V projections) runs here.
//
// Design (B200-first):
//  * persistent grid (<= #free SMs), static tile walk with N fastest so the
//    CTAs working on one 128-row A block run together and share it in L2;
//  * warp 0: TMA producer (128B-swizzled 128x64 A and BNx64 W tiles into an
//    S-stage smem ring, mbarrier full/empty);
//  * warp 1: allocates TMEM and issues tcgen05.mma (M=128, N=BN, K=16) from
//    one elected lane; tcgen05.commit frees smem stages / publishes an
//    accumulator;
//  * warps 2-9: epilogue — tcgen05.ld of the fp32 accumulator (each warp owns
//    its 32-lane TMEM quarter), fused bias / GELU / adaLN-gated residual /
//    K-V-slot scatter, direct global stores;
//  * the accumulator is double-buffered in TMEM (2 x BN columns) so the
//    epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "../kernels.h"

namespace stadi {

namespace {

constexpr int GBM = 128, GBK = 64;

constexpr int EPI_LD = 33;                       // staging row stride (floats, bank-free)
// STADI_GEMM_EPI_WARPS (compile time): 8 = two per TMEM lane quarter (column halves); 4 =
// one per quarter (6 warps per CTA, so the per-SM-sub-partition register budget allows
// 256 registers per thread instead of 168: no epilogue spills)
#ifndef STADI_GEMM_EPI_WARPS
#define STADI_GEMM_EPI_WARPS 8
#endif
constexpr int EPI_WARPS = STADI_GEMM_EPI_WARPS;
constexpr int EPI_STEP = EPI_WARPS / 4;            // chunk stride of one epilogue warp
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;
constexpr int EPI_SMEM = EPI_WARPS * 32 * EPI_LD * 4;  // per warp 32 x 32 fp32 staging

// MC: 1 = one CTA per tile; 2 = CTA pair, each CTA its own 128-row tile, the W tile
// loaded half by each CTA and multicast to both; 3 = CTA pair running ONE
// M = 256 tcgen05.mma (cta_group::2) issued by the leader: each CTA stages its
// own 128 A rows and HALF of the W tile, so per-SM shared-memory traffic per
// MMA is halved.
template <int BN, int MC = 1>
struct GemmCfg {
  static constexpr int A_BYTES = GBM * GBK * 2;              // 16 KB
  static constexpr int B_BYTES = (MC == 3 ? BN / 2 : BN) * GBK * 2;  // per CTA
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int RING = 227 * 1024 - EPI_SMEM - 1024 /*align*/ - 256 /*barriers*/;
  static constexpr int STAGES = RING / STAGE > 8 ? 8 : RING / STAGE;
  static constexpr int TMEM_COLS = (2 * BN <= 128) ? 128 : (2 * BN <= 256 ? 256 : 512);
  static constexpr int SMEM = STAGES * STAGE + EPI_SMEM + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(SMEM <= 227 * 1024 && STAGES >= 2, "GEMM shared memory");
};

// Epilogue of two adjacent columns (col even) of one row, vectorised stores.
// Split in two so a warp can issue the global reads of all its rows first (the
// residual of RES / GATED_RES / CONV is read-modify-write in HBM: issuing the 16
// loads of a chunk back to back hides their latency behind each other).
struct EpiIn {
  float2 r;  // residual (the only operand streamed from HBM)
};
template <int EPI>
__device__ __forceinline__ EpiIn epi_load(const EpiParams &p, int row, int col) {
  EpiIn in;
  in.r = make_float2(0.f, 0.f);
  if constexpr (EPI == EPI_GATED_RES || EPI == EPI_RES || EPI == EPI_CONV) {
    if (p.res) in.r = *reinterpret_cast<const float2 *>(p.res + (long)row * p.ldr + col);
  }
  return in;
}
// Per-chunk constants of a lane's column pair: bias and the B (<= 2) gate rows,
// loaded once per 32-column chunk instead of once per row.
struct EpiCol {
  float2 b, g0, g1;  // bias; gate rows of batch 0 / 1 (no dynamic indexing: registers)
};
template <int EPI>
__device__ __forceinline__ EpiCol epi_col(const EpiParams &p, int col) {
  EpiCol c;
  c.b = p.bias ? *reinterpret_cast<const float2 *>(p.bias + col) : make_float2(0.f, 0.f);
  c.g0 = c.g1 = make_float2(0.f, 0.f);
  if constexpr (EPI == EPI_GATED_RES || EPI == EPI_CONV) {
    if (p.gate) {
      c.g0 = *reinterpret_cast<const float2 *>(p.gate + col);
      c.g1 = p.B > 1 ? *reinterpret_cast<const float2 *>(p.gate + p.gate_bstride + col) : c.g0;
    }
  }
  return c;
}
__device__ __forceinline__ float gelu_tanh_fast(float x) {  // MUFU.TANH
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.7978845608028654f * (x + 0.044715f * x * x * x)));
  return 0.5f * x * (1.f + t);
}
template <int EPI>
__device__ __forceinline__ void epi_finish(const EpiParams &p, int row, int col, float v0,
                                           float v1, const EpiIn &in, const EpiCol &cc) {
  v0 += cc.b.x;
  v1 += cc.b.y;
  const float2 g = (row % p.B) ? cc.g1 : cc.g0;
  if constexpr (EPI == EPI_STORE || EPI == EPI_GELU) {
    if (EPI == EPI_GELU) {
      v0 = gelu_tanh_fast(v0);
      v1 = gelu_tanh_fast(v1);
    }
    *reinterpret_cast<__nv_bfloat162 *>(reinterpret_cast<bf16 *>(p.out) + (long)row * p.ldo +
                                        col) = __floats2bfloat162_rn(v0, v1);
  } else if constexpr (EPI == EPI_F32 || EPI == EPI_CONV) {
    if constexpr (EPI == EPI_CONV) {
      v0 += g.x + in.r.x;
      v1 += g.y + in.r.y;
    }
    *reinterpret_cast<float2 *>(reinterpret_cast<float *>(p.out) + (long)row * p.ldo + col) =
        make_float2(v0, v1);
  } else if constexpr (EPI == EPI_GATED_RES) {
    *reinterpret_cast<float2 *>(p.res + (long)row * p.ldr + col) =
        make_float2(in.r.x + g.x * v0, in.r.y + g.y * v1);
  } else if constexpr (EPI == EPI_RES) {
    *reinterpret_cast<float2 *>(p.res + (long)row * p.ldr + col) =
        make_float2(in.r.x + v0, in.r.y + v1);
  } else if constexpr (EPI == EPI_GEGLU) {
    reinterpret_cast<bf16 *>(p.out)[(long)row * p.ldo + col / 2] =
        __float2bfloat16_rn(v0 * gelu_erf(v1));
  } else if constexpr (EPI == EPI_QKV) {
    const __nv_bfloat162 t = __floats2bfloat162_rn(v0, v1);
    if (col < p.d) {
      *reinterpret_cast<__nv_bfloat162 *>(reinterpret_cast<bf16 *>(p.q) + (long)row * p.d + col) =
          t;
    } else {
      const long off = (p.kv_row0 + row) * 2L * p.d + (col - p.d);
      *reinterpret_cast<__nv_bfloat162 *>(reinterpret_cast<bf16 *>(p.kv_a) + off) = t;
      if (p.kv_b) *reinterpret_cast<__nv_bfloat162 *>(reinterpret_cast<bf16 *>(p.kv_b) + off) = t;
      for (int k = 0; k < p.n_kv_peer; ++k)  // IPC peers (P2P stores over NVLink)
        *reinterpret_cast<__nv_bfloat162 *>(reinterpret_cast<bf16 *>(p.kv_peer[k]) + off) = t;
    }
  }
}

// Implicit 3x3 convolution (AM == 1): the A operand is not materialised; for
// K block kb = (tap, 64-channel chunk) the producer TMA-loads the 128 output
// rows' input pixels shifted by the tap straight from the halo-padded NHWC
// buffer P [h+2, W+2, B, C] with a 3-D box (64 ch, min(W B, 128) pixel-batch
// rows, 128 / (W B) image rows): exactly the K-major 128B-swizzled A tile.
struct ConvGeo {
  int W, B, C;  // band width, batch, input channels (C % 64 == 0)
};

template <int BN, int EPI, int MC, int AM>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   int M, int N, int K, EpiParams ep, ConvGeo cg, int ksplit) {
  using C = GemmCfg<BN, MC>;
  constexpr int NCL = MC == 1 ? 1 : 2;  // cluster size
  constexpr bool PAIR = MC == 3;        // cta_group::2 MMA
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + C::STAGES * C::A_BYTES;
  float *stg_all = reinterpret_cast<float *>(smem + C::STAGES * C::STAGE);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE + EPI_SMEM);
  uint64_t *full = bars, *empty = bars + C::STAGES;
  uint64_t *tfull = bars + 2 * C::STAGES, *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles_n = N / BN, tiles_m = (M + GBM - 1) / GBM;
  const int nkb = K / GBK;
  // tile walk: NCL row tiles (one per cluster CTA) per work item, N fastest
  const int crank = NCL == 2 ? (int)cluster_ctarank() : 0;
  // split-K (ksplit > 1): item = (tile, split); split sp accumulates k blocks
  // [sp nkb / ksplit, (sp + 1) nkb / ksplit) and stores an fp32 partial tile into
  // ep.ws[sp]; splitk_reduce_kernel sums the partials in split order (deterministic)
  // and runs the epilogue
  const int n_items = ((tiles_m + NCL - 1) / NCL) * tiles_n * ksplit;
  const int item0 = blockIdx.x / NCL, item_step = gridDim.x / NCL;
  auto tile_of = [&](int item, int *mb, int *nb) {
    const int t = item / ksplit;
    *mb = (t / tiles_n) * NCL + crank;
    *nb = t % tiles_n;
  };
  auto k_range = [&](int item, int *kb0, int *kb1) {
    const int sp = item % ksplit;
    *kb0 = (int)((long)sp * nkb / ksplit);
    *kb1 = (int)((long)(sp + 1) * nkb / ksplit);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC == 2 ? 2 : 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], (PAIR ? 2 : 1) * EPI_WARPS);  // one arrive per epilogue warp (of the pair)
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_cg2(tmem_slot, C::TMEM_COLS);
    else tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if (NCL == 2) cluster_sync();  // partner's barriers initialised before any multicast
  pdl_wait();                    // the predecessor's outputs (A, residual) are complete
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (int item = item0; item < n_items; item += item_step) {
        int mb, nb, kb0, kb1;
        tile_of(item, &mb, &nb);
        k_range(item, &kb0, &kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          if (!PAIR || crank == 0) mbar_expect_tx(&full[s], (PAIR ? 2 : 1) * C::STAGE);
          if constexpr (AM == 1) {
            const int cpb = cg.C / GBK, tap = kb / cpb, c0 = (kb % cpb) * GBK;
            const int p0 = mb * (GBM / cg.B);  // first output pixel of the tile
            if constexpr (PAIR)
              tma_load_3d_cg2(&tmA, sA + s * C::A_BYTES, &full[s], c0,
                              (p0 % cg.W + tap % 3) * cg.B, p0 / cg.W + tap / 3);
            else
              tma_load_3d(&tmA, sA + s * C::A_BYTES, &full[s], c0,
                          (p0 % cg.W + tap % 3) * cg.B, p0 / cg.W + tap / 3);
          } else if constexpr (AM == 2) {  // stride 2: every other pixel / row of P
            const int cpb = cg.C / GBK, tap = kb / cpb, c0 = (kb % cpb) * GBK;
            const int wo = cg.W / 2, p0 = mb * (GBM / cg.B);
            const int x = 2 * (p0 % wo) + tap % 3, y = 2 * (p0 / wo) + tap / 3;
            if constexpr (PAIR)
              tma_load_4d_cg2(&tmA, sA + s * C::A_BYTES, &full[s], c0, 0, x, y);
            else
              tma_load_4d(&tmA, sA + s * C::A_BYTES, &full[s], c0, 0, x, y);
          } else if constexpr (PAIR) {
            tma_load_2d_cg2(&tmA, sA + s * C::A_BYTES, &full[s], kb * GBK, mb * GBM);
          } else {
            tma_load_2d(&tmA, sA + s * C::A_BYTES, &full[s], kb * GBK, mb * GBM);
          }
          if constexpr (PAIR)
            tma_load_2d_cg2(&tmB, sB + s * C::B_BYTES, &full[s], kb * GBK,
                            nb * BN + crank * (BN / 2));
          else if constexpr (MC == 2)
            tma_load_2d_mc(&tmB, sB + s * C::B_BYTES + crank * (C::B_BYTES / 2), &full[s],
                           kb * GBK, nb * BN + crank * (BN / 2), (uint16_t)0x3);
          else
            tma_load_2d(&tmB, sB + s * C::B_BYTES, &full[s], kb * GBK, nb * BN);
          if (++s == C::STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (!PAIR || crank == 0) {  // ---------------- MMA issuer (pair: leader), whole warp
      // warp-collective issue (one elected lane in the asm): descriptors stay in
      // uniform registers -- see umma_bf16_w
      constexpr uint32_t idesc = umma_idesc_bf16(PAIR ? 2 * GBM : GBM, BN, 0, 0);
      const uint64_t adesc0 = umma_desc(smem_u32(sA), 16, 1024, SWZ_128B);
      const uint64_t bdesc0 = umma_desc(smem_u32(sB), 16, 1024, SWZ_128B);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int item = item0; item < n_items; item += item_step, ++it) {
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem + acc * BN;
        int kb0, kb1;
        k_range(item, &kb0, &kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          // stage descriptors = stage-0 descriptors + the stage's 16-byte offset
          const uint64_t ad = adesc0 + (uint64_t)((uint32_t)s * (uint32_t)(C::A_BYTES >> 4));
          const uint64_t bd = bdesc0 + (uint64_t)((uint32_t)s * (uint32_t)(C::B_BYTES >> 4));
#pragma unroll
          for (int k = 0; k < GBK / 16; ++k) {
            if constexpr (PAIR) umma_bf16_cg2_w(dtm, ad + 2 * k, bd + 2 * k, idesc, (kb - kb0) | k);
            else umma_bf16_w(dtm, ad + 2 * k, bd + 2 * k, idesc, (kb - kb0) | k);
          }
          if constexpr (PAIR) umma_commit_cg2_w(&empty[s]);
          else if constexpr (MC == 2) umma_commit_mc_w(&empty[s], (uint16_t)0x3);
          else umma_commit_w(&empty[s]);
          if (++s == C::STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if constexpr (PAIR) umma_commit_cg2_w(&tfull[acc]);
        else umma_commit_w(&tfull[acc]);
      }
    }
  } else {  // ---------------------------- epilogue warps 2..9
    const int qd = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - 2) / 4;  // 32-column chunks half, half + EPI_STEP, ... of the tile
    constexpr int NCHUNK = BN / 32;
    static_assert(BN % 32 == 0, "epilogue chunks");
    // residual RMW epilogues use 16-byte accesses when every operand row is 16-B aligned
    const bool vec4 = ep.res_vec4 && ep.res != nullptr &&
                      ((reinterpret_cast<uintptr_t>(ep.res) | reinterpret_cast<uintptr_t>(ep.bias) |
                        reinterpret_cast<uintptr_t>(ep.gate) | (uintptr_t)ep.ldr * 4u |
                        (uintptr_t)ep.gate_bstride * 4u) & 15u) == 0 &&
                      (EPI != EPI_CONV ||
                       ((reinterpret_cast<uintptr_t>(ep.out) | (uintptr_t)ep.ldo * 4u) & 15u) == 0);
    // plain-store epilogues: 8-byte (bf16) / 16-byte (fp32) output rows, 16-byte bias
    const bool vec4o =
        EPI == EPI_QKV
            ? ep.res_vec4 && (reinterpret_cast<uintptr_t>(ep.bias) & 15u) == 0 &&
                  ((reinterpret_cast<uintptr_t>(ep.q) | reinterpret_cast<uintptr_t>(ep.kv_a) |
                    reinterpret_cast<uintptr_t>(ep.kv_b) | (uintptr_t)ep.d * 2u) & 7u) == 0
            : ep.res_vec4 && ep.out != nullptr && (reinterpret_cast<uintptr_t>(ep.bias) & 15u) == 0 &&
                  ((reinterpret_cast<uintptr_t>(ep.out) |
                    (uintptr_t)ep.ldo * (EPI == EPI_F32 ? 4u : 2u)) &
                   (EPI == EPI_F32 ? 15u : (EPI == EPI_GEGLU ? 3u : 7u))) == 0;
    int it = 0;
    for (int item = item0; item < n_items; item += item_step, ++it) {
      int mb, nb;
      tile_of(item, &mb, &nb);
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const int row0 = mb * GBM + qd * 32;
      if constexpr (EPI == EPI_GATED_RES || EPI == EPI_RES || EPI == EPI_CONV) {
        // the fp32 residual is the epilogue's only HBM read: pull this warp's
        // rows x chunks (one 128-B line per row and 32-column chunk) into L2
        // while the tile's MMAs still run, so the epilogue reads hit L2
        if (ep.res_prefetch && ep.res && ksplit == 1 && row0 + lane < M) {
          const float *rp = ep.res + (long)(row0 + lane) * ep.ldr + nb * BN;
#pragma unroll 1
          for (int ch = half; ch < NCHUNK; ch += EPI_STEP)
            asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(rp + 32 * ch));
        }
      }
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16) + acc * BN;
      float *stg = stg_all + (warp - 2) * 32 * EPI_LD;
#pragma unroll 1
      for (int ch = half; ch < NCHUNK; ch += EPI_STEP) {
        const int c0 = 32 * ch;
        // TMEM -> registers (lane = row) -> smem, then coalesced: lanes cover
        // 16 column pairs of two rows per step
        float v[32];
        tmem_ld32(tbase + c0, v);
        if (ch + EPI_STEP >= NCHUNK) {  // this warp's chunks read: release the accumulator
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (PAIR) mbar_arrive_cluster(&tempty[acc], 0);  // the leader's
            else mbar_arrive(&tempty[acc]);
          }
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) stg[lane * EPI_LD + i] = v[i];
        __syncwarp();
        const int cc = 2 * (lane & 15), col = nb * BN + c0 + cc;
        if (ksplit > 1) {  // fp32 partial tile of split `item % ksplit`
          float *wsp = ep.ws + (long)(item % ksplit) * M * N;
#pragma unroll
          for (int it = 0; it < 16; ++it) {
            const int r = 2 * it + (lane >> 4);
            if (row0 + r < M)
              *reinterpret_cast<float2 *>(wsp + (long)(row0 + r) * N + col) =
                  make_float2(stg[r * EPI_LD + cc], stg[r * EPI_LD + cc + 1]);
          }
          __syncwarp();
          continue;
        }
        if constexpr (EPI == EPI_GATED_RES || EPI == EPI_RES || EPI == EPI_CONV) {
          if (vec4) {  // 16-byte residual RMW: 8 lanes per row, 4 rows per step
            const int c4 = 4 * (lane & 7), col4 = nb * BN + c0 + c4;
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 b4 = ep.bias ? *reinterpret_cast<const float4 *>(ep.bias + col4) : z4;
            float4 g0 = z4, g1 = z4;
            if constexpr (EPI == EPI_GATED_RES || EPI == EPI_CONV) {
              if (ep.gate) {
                g0 = *reinterpret_cast<const float4 *>(ep.gate + col4);
                g1 = ep.B > 1 ? *reinterpret_cast<const float4 *>(ep.gate + ep.gate_bstride + col4)
                              : g0;
              }
            }
            float4 rin[8];
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int row = row0 + 4 * it + (lane >> 3);
              if (row < M) rin[it] = *reinterpret_cast<const float4 *>(ep.res + (long)row * ep.ldr + col4);
            }
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int r = 4 * it + (lane >> 3), row = row0 + r;
              if (row >= M) continue;
              const float *sv = stg + r * EPI_LD + c4;
              const float4 v = make_float4(sv[0] + b4.x, sv[1] + b4.y, sv[2] + b4.z, sv[3] + b4.w);
              float4 o;  // the same expressions (and FMA contraction) as epi_finish
              if constexpr (EPI == EPI_GATED_RES) {
                const float4 g = (row % ep.B) ? g1 : g0;
                o = make_float4(rin[it].x + g.x * v.x, rin[it].y + g.y * v.y,
                                rin[it].z + g.z * v.z, rin[it].w + g.w * v.w);
              } else if constexpr (EPI == EPI_CONV) {  // v += (time bias + residual)
                const float4 g = (row % ep.B) ? g1 : g0;
                o = make_float4(v.x + (g.x + rin[it].x), v.y + (g.y + rin[it].y),
                                v.z + (g.z + rin[it].z), v.w + (g.w + rin[it].w));
                *reinterpret_cast<float4 *>(reinterpret_cast<float *>(ep.out) + (long)row * ep.ldo +
                                            col4) = o;
                continue;
              } else {
                o = make_float4(rin[it].x + v.x, rin[it].y + v.y, rin[it].z + v.z, rin[it].w + v.w);
              }
              *reinterpret_cast<float4 *>(ep.res + (long)row * ep.ldr + col4) = o;
            }
            __syncwarp();
            continue;
          }
        }
        if constexpr (EPI == EPI_STORE || EPI == EPI_GELU || EPI == EPI_F32 || EPI == EPI_QKV ||
                      EPI == EPI_GEGLU) {
          if (vec4o) {  // 8-byte bf16 / 16-byte fp32 stores: 8 lanes per row, 4 rows per step
            const int c4 = 4 * (lane & 7), col4 = nb * BN + c0 + c4;
            const float4 b4 = ep.bias ? *reinterpret_cast<const float4 *>(ep.bias + col4)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int r = 4 * it + (lane >> 3), row = row0 + r;
              if (row >= M) continue;
              const float *sv = stg + r * EPI_LD + c4;
              float v0 = sv[0] + b4.x, v1 = sv[1] + b4.y, v2 = sv[2] + b4.z, v3 = sv[3] + b4.w;
              if constexpr (EPI == EPI_GEGLU) {  // (a, g) pairs -> two outputs, one 4-byte store
                *reinterpret_cast<__nv_bfloat162 *>(reinterpret_cast<bf16 *>(ep.out) +
                                                    (long)row * ep.ldo + col4 / 2) =
                    __floats2bfloat162_rn(v0 * gelu_erf(v1), v2 * gelu_erf(v3));
              } else if constexpr (EPI == EPI_F32) {
                *reinterpret_cast<float4 *>(reinterpret_cast<float *>(ep.out) + (long)row * ep.ldo +
                                            col4) = make_float4(v0, v1, v2, v3);
              } else {
                if constexpr (EPI == EPI_GELU) {
                  v0 = gelu_tanh_fast(v0);
                  v1 = gelu_tanh_fast(v1);
                  v2 = gelu_tanh_fast(v2);
                  v3 = gelu_tanh_fast(v3);
                }
                const __nv_bfloat162 lo = __floats2bfloat162_rn(v0, v1),
                                     hi = __floats2bfloat162_rn(v2, v3);
                uint2 pk;
                pk.x = *reinterpret_cast<const uint32_t *>(&lo);
                pk.y = *reinterpret_cast<const uint32_t *>(&hi);
                if constexpr (EPI == EPI_QKV) {  // d % 4 == 0: a 4-column group never straddles q | kv
                  if (col4 < ep.d) {
                    *reinterpret_cast<uint2 *>(reinterpret_cast<bf16 *>(ep.q) + (long)row * ep.d + col4) = pk;
                  } else {
                    const long off = (ep.kv_row0 + row) * 2L * ep.d + (col4 - ep.d);
                    *reinterpret_cast<uint2 *>(reinterpret_cast<bf16 *>(ep.kv_a) + off) = pk;
                    if (ep.kv_b) *reinterpret_cast<uint2 *>(reinterpret_cast<bf16 *>(ep.kv_b) + off) = pk;
                    for (int k = 0; k < ep.n_kv_peer; ++k)  // IPC peers (P2P stores)
                      *reinterpret_cast<uint2 *>(reinterpret_cast<bf16 *>(ep.kv_peer[k]) + off) = pk;
                  }
                } else {
                  *reinterpret_cast<uint2 *>(reinterpret_cast<bf16 *>(ep.out) + (long)row * ep.ldo +
                                             col4) = pk;
                }
              }
            }
            __syncwarp();
            continue;
          }
        }
        const EpiCol ecol = epi_col<EPI>(ep, col);
        EpiIn in[16];
#pragma unroll
        for (int it = 0; it < 16; ++it) {  // all global reads of the chunk in flight
          const int row = row0 + 2 * it + (lane >> 4);
          if (row < M) in[it] = epi_load<EPI>(ep, row, col);
        }
#pragma unroll
        for (int it = 0; it < 16; ++it) {
          const int r = 2 * it + (lane >> 4);
          if (row0 + r < M)
            epi_finish<EPI>(ep, row0 + r, col, stg[r * EPI_LD + cc], stg[r * EPI_LD + cc + 1],
                            in[it], ecol);
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (NCL == 2) cluster_sync();  // no CTA leaves while its partner may still signal it
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_cg2(tmem, C::TMEM_COLS);
    else tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// Split-K epilogue: sum the ksplit fp32 partial tiles in split order (the same
// order every run: deterministic), then the GEMM epilogue on the column pair.
template <int EPI>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(int M, int N, int ksplit, EpiParams ep) {
  pdl_wait();
  const long quads = (long)M * (N / 4);
  const long plane = (long)M * N;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < quads;
       i += (long)gridDim.x * blockDim.x) {
    const int row = (int)(i / (N / 4)), col = 4 * (int)(i % (N / 4));
    const float *w = ep.ws + (long)row * N + col;
    float4 a = *reinterpret_cast<const float4 *>(w);
    for (int sp = 1; sp < ksplit; ++sp) {
      const float4 b = *reinterpret_cast<const float4 *>(w + sp * plane);
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    const EpiCol c0 = epi_col<EPI>(ep, col), c1 = epi_col<EPI>(ep, col + 2);
    const EpiIn i0 = epi_load<EPI>(ep, row, col), i1 = epi_load<EPI>(ep, row, col + 2);
    epi_finish<EPI>(ep, row, col, a.x, a.y, i0, c0);
    epi_finish<EPI>(ep, row, col + 2, a.z, a.w, i1, c1);
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                              const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                              const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

}  // namespace

// Exported for the attention kernel too.  estr: per-dimension element (traversal)
// strides (NULL = all 1): TMA then loads ceil(box[i] / estr[i]) elements along i.
bool make_tmap(CUtensorMap *m, const void *base, int rank, const uint64_t *dims,
               const uint64_t *strides_bytes, const uint32_t *box, CUtensorMapSwizzle swz,
               const uint32_t *estr = nullptr) {
  EncodeFn fn = get_encode();
  if (!fn) return false;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = estr ? estr[i] : 1;
  }
  for (int i = 0; i < rank - 1; ++i) st[i] = strides_bytes[i];
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void *>(base), d, st, b,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {
constexpr int NCL_OF(int mc) { return mc == 1 ? 1 : 2; }
// STADI_SPLITK=0 disables split-K (A/B comparisons).
// STADI_RES_PREFETCH=0 disables the residual L2 prefetch (A/B comparisons).
bool res_prefetch_enabled() {
  static const int v = [] {
    const char *e = getenv("STADI_RES_PREFETCH");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v != 0;
}
// STADI_RES_VEC4=0 keeps the 8-byte residual epilogue (A/B comparisons).
bool res_vec4_enabled() {
  static const int v = [] {
    const char *e = getenv("STADI_RES_VEC4");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v != 0;
}
bool splitk_disabled() {
  static const int v = [] {
    const char *e = getenv("STADI_SPLITK");
    return (e && e[0] == '0') ? 1 : 0;
  }();
  return v != 0;
}
template <int BN, int EPI, int MC, int AM>
cudaError_t launch_gemm(const bf16 *A, const bf16 *W, int M, int N, int K, const EpiParams &ep,
                        int max_ctas, const ConvGeo &cg, int conv_h, int ksplit, cudaStream_t s) {
  if (ksplit > 1 && (!ep.ws || (long)ksplit * M * N > ep.ws_elems)) return cudaErrorInvalidValue;
  using C = GemmCfg<BN, MC>;
  constexpr int NCL = MC == 1 ? 1 : 2;
  CUtensorMap ta, tb;
  bool ok;
  if constexpr (AM == 1) {  // P [h+2, (W+2) B, C]
    const int wb = cg.W * cg.B;
    const uint64_t da[3] = {(uint64_t)cg.C, (uint64_t)(cg.W + 2) * cg.B, (uint64_t)conv_h + 2};
    const uint64_t sa[2] = {(uint64_t)cg.C * 2, (uint64_t)(cg.W + 2) * cg.B * cg.C * 2};
    const uint32_t ba[3] = {GBK, (uint32_t)std::min(wb, GBM), (uint32_t)std::max(1, GBM / wb)};
    ok = make_tmap(&ta, A, 3, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B);
  } else if constexpr (AM == 2) {  // P [h+2, W+2, B, C], every other pixel / row
    const int wob = cg.W / 2 * cg.B;
    const uint64_t da[4] = {(uint64_t)cg.C, (uint64_t)cg.B, (uint64_t)cg.W + 2,
                            (uint64_t)conv_h + 2};
    const uint64_t sa[3] = {(uint64_t)cg.C * 2, (uint64_t)cg.B * cg.C * 2,
                            (uint64_t)(cg.W + 2) * cg.B * cg.C * 2};
    const uint32_t ba[4] = {GBK, (uint32_t)cg.B, (uint32_t)(2 * std::min(wob, GBM) / cg.B),
                            (uint32_t)(2 * std::max(1, GBM / wob))};
    const uint32_t es[4] = {1, 1, 2, 2};
    ok = make_tmap(&ta, A, 4, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B, es);
  } else {
    const uint64_t da[2] = {(uint64_t)K, (uint64_t)M}, sa[1] = {(uint64_t)K * 2};
    const uint32_t ba[2] = {GBK, GBM};
    ok = make_tmap(&ta, A, 2, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  const uint64_t db[2] = {(uint64_t)K, (uint64_t)N}, sb[1] = {(uint64_t)K * 2};
  const uint32_t bb[2] = {GBK, (uint32_t)(BN / NCL)};
  if (!ok || !make_tmap(&tb, W, 2, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  static bool attr_set = false;  // per template instance
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, EPI, MC, AM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int items = ((M + GBM - 1) / GBM + NCL - 1) / NCL * (N / BN) * ksplit;
  int grid = std::min(items * NCL, max_ctas / NCL * NCL);
  if (grid < NCL) grid = NCL;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = NCL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  EpiParams epk = ep;
  epk.res_prefetch = res_prefetch_enabled() ? 1 : 0;
  epk.res_vec4 = res_vec4_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_kernel<BN, EPI, MC, AM>, ta, tb, M, N, K, epk,
                                     cg, ksplit);
  ++g_launches;
  if (e != cudaSuccess) return e;
  if (ksplit > 1) {
    const long quads = (long)M * (N / 4);
    const int rb = (int)std::min<long>((quads + 255) / 256, 148L * 8);
    cudaError_t e2 = launch_pdl(splitk_reduce_kernel<EPI>, dim3(rb), dim3(256), 0, s, M, N, ksplit, ep);
    if (e2 != cudaSuccess) return e2;
    ++g_launches;
  }
  return cudaGetLastError();
}

template <int BN, int MC>
cudaError_t dispatch_epi(const bf16 *A, const bf16 *W, int M, int N, int K, int epi,
                         const EpiParams &ep, int max_ctas, int ks, cudaStream_t s) {
  const ConvGeo g{0, 0, 0};
  switch (epi) {
    case EPI_STORE: return launch_gemm<BN, EPI_STORE, MC, 0>(A, W, M, N, K, ep, max_ctas, g, 0, ks, s);
    case EPI_GELU: return launch_gemm<BN, EPI_GELU, MC, 0>(A, W, M, N, K, ep, max_ctas, g, 0, ks, s);
    case EPI_GATED_RES:
      return launch_gemm<BN, EPI_GATED_RES, MC, 0>(A, W, M, N, K, ep, max_ctas, g, 0, ks, s);
    case EPI_RES: return launch_gemm<BN, EPI_RES, MC, 0>(A, W, M, N, K, ep, max_ctas, g, 0, ks, s);
    case EPI_QKV: return launch_gemm<BN, EPI_QKV, MC, 0>(A, W, M, N, K, ep, max_ctas, g, 0, ks, s);
    case EPI_F32: return launch_gemm<BN, EPI_F32, MC, 0>(A, W, M, N, K, ep, max_ctas, g, 0, ks, s);
    case EPI_CONV: return launch_gemm<BN, EPI_CONV, MC, 0>(A, W, M, N, K, ep, max_ctas, g, 0, ks, s);
    case EPI_GEGLU: return launch_gemm<BN, EPI_GEGLU, MC, 0>(A, W, M, N, K, ep, max_ctas, g, 0, ks, s);
  }
  return cudaErrorInvalidValue;
}
template <int BN>
cudaError_t dispatch_mc(const bf16 *A, const bf16 *W, int M, int N, int K, int epi,
                        const EpiParams &ep, int max_ctas, int mc, int ks, cudaStream_t s) {
  if (mc == 3) return dispatch_epi<BN, 3>(A, W, M, N, K, epi, ep, max_ctas, ks, s);
  if (mc == 2) return dispatch_epi<BN, 2>(A, W, M, N, K, epi, ep, max_ctas, ks, s);
  return dispatch_epi<BN, 1>(A, W, M, N, K, epi, ep, max_ctas, ks, s);
}
template <int BN, int MC>
cudaError_t dispatch_conv(const bf16 *P, const bf16 *W, int h, const ConvGeo &g, int N, int epi,
                          const EpiParams &ep, int max_ctas, int ks, int mode, cudaStream_t s) {
  const int K = 9 * g.C;
  if (mode == 1) {  // stride 2: (h / 2) x (W / 2) outputs
    const int M = h / 2 * (g.W / 2) * g.B;
    if (epi == EPI_CONV)
      return launch_gemm<BN, EPI_CONV, MC, 2>(P, W, M, N, K, ep, max_ctas, g, h, ks, s);
    if (epi == EPI_F32)
      return launch_gemm<BN, EPI_F32, MC, 2>(P, W, M, N, K, ep, max_ctas, g, h, ks, s);
    return cudaErrorInvalidValue;
  }
  const int M = h * g.W * g.B;
  if (epi == EPI_CONV)
    return launch_gemm<BN, EPI_CONV, MC, 1>(P, W, M, N, K, ep, max_ctas, g, h, ks, s);
  if (epi == EPI_F32)
    return launch_gemm<BN, EPI_F32, MC, 1>(P, W, M, N, K, ep, max_ctas, g, h, ks, s);
  return cudaErrorInvalidValue;
}
}  // namespace

// Tile width BN and K split of one GEMM from a small cost model of B200 (clocks of
// one SM): a CTA's 64-deep k block costs max(2 BN MMA clocks (M = 128 rows per
// CTA), its operand bytes / the per-SM share of the ~6300 B/clk chip L2 limit)
// (A 16 KB + W BN x 128 B, or half of W when a CTA pair shares it), plus ~1500
// clocks of fill / epilogue per work item; waves of the persistent grid; split-K
// adds the fp32 partial round trip through L2/HBM and a reduce launch.
struct GemmPlan {
  int bn, ks;
};
// STADI_GEMM_L2=<bytes per clock>: the cost model's chip L2 bandwidth (default 12600:
// measured in-step, C3 334 -> 317 ms and C4 1232 -> 1180 ms / image against 6300).
double gemm_l2_bw() {
  static const double v = [] {
    const char *e = getenv("STADI_GEMM_L2");
    const double x = e ? atof(e) : 0.0;
    return x > 0 ? x : 12600.0;
  }();
  return v;
}
// STADI_GEMM_BN=<64|128|160|192|256>: force the tile width where it divides N (A/B only).
int gemm_forced_bn() {
  static const int v = [] {
    const char *e = getenv("STADI_GEMM_BN");
    return e ? atoi(e) : 0;
  }();
  return v;
}
GemmPlan plan_gemm(int M, int N, int K, int max_ctas, int mc, long ws_elems) {
  const int tm = (M + GBM - 1) / GBM, nkb = K / GBK;
  const double L2 = gemm_l2_bw();
  if (const int fb = gemm_forced_bn(); fb && N % fb == 0 &&
      (fb == 64 || fb == 128 || fb == 160 || fb == 192 || fb == 256))
    return GemmPlan{fb, 1};
  const int ncl = mc == 1 ? 1 : 2;
  const int tmr = (tm + ncl - 1) / ncl * ncl;
  const int cands[5] = {256, 192, 160, 128, 64};
  GemmPlan best{64, 1};
  double best_t = -1;
  for (int bn : cands) {
    if (N % bn) continue;
    const double wbytes = (mc == 1 ? 128.0 : 64.0) * bn;
    const double per_kb = std::max(2.0 * bn, (16384.0 + wbytes) / (L2 / max_ctas));
    for (int ks = 1; ks <= 16; ++ks) {
      if (ks > 1 && (nkb / ks < 8 || (long)ks * M * N > ws_elems || splitk_disabled())) break;
      const long ctas = (long)tmr * (N / bn) * ks;
      const long waves = (ctas + max_ctas - 1) / max_ctas;
      const long per_cta = (ctas + waves - 1) / waves;  // CTAs of a wave, sharing L2
      const double kb = (double)nkb / ks;
      const double l2 = kb * (16384.0 + wbytes) * per_cta / L2;
      double t = waves * std::max(kb * 2.0 * bn + 1500.0, l2 + 1500.0);
      if (ks > 1) t += (ks + 2.0) * M * N * 4.0 / 3300.0 + 4000.0;
      if (best_t < 0 || t < best_t * 0.97) {  // prefer the earlier (wider, unsplit) option
        best_t = t;
        best = {bn, ks};
      }
    }
  }
  return best;
}

// CTA-pair mode of the GEMMs with >= 4 row tiles (see GemmCfg).  Default (measured
// on B200, tools/kbench.py gemm): the cta_group::2 M = 256 MMA, except for the
// fp32 residual read-modify-write epilogues, whose HBM-bound epilogue prefers
// two independent 128-row tiles with a multicast W tile (C5 out-proj 654 vs 613
// TFLOP/s; 8192^3 1342 vs 1278 the other way).  STADI_GEMM_MC=0 / 2 / 3 forces
// single-CTA tiles / multicast pairs / the cta_group::2 MMA (A/B comparisons).
bool pdl_enabled() {
  static const bool v = [] {
    const char *e = getenv("STADI_PDL");
    return !(e && e[0] == '0');
  }();
  return v;
}

int gemm_pair_mode() {
  static const int v = [] {
    const char *e = getenv("STADI_GEMM_MC");
    if (e && e[0] == '0') return 1;
    if (e && e[0] == '2') return 2;
    if (e && e[0] == '3') return 3;
    return 0;
  }();
  return v;
}
int device_sms() {
  static const int v = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return v;
}
int pair_mode_for(int tm, int max_ctas, int epi, int K) {
  // Fewer CTAs than SMs means the occupancy emulator holds the rest: launch
  // single-CTA tiles, free of cluster-placement constraints on a partly held GPU
  // (measured on B200 with the C2 / C5 shapes at 20-60%: same speed as CTA pairs;
  // STADI_GEMM_MC overrides).
  if (tm < 4 || max_ctas < 2) return 1;
  if (gemm_pair_mode()) return gemm_pair_mode();
  if (max_ctas < device_sms()) return 1;
  // residual RMW epilogues: multicast pairs while the epilogue's HBM traffic rules
  // (K = 1152 out-proj 143 vs 154 us), the cta_group::2 MMA once the K loop does
  // (K = 4608 fc2 314 vs 320 us)
  return ((epi == EPI_GATED_RES || epi == EPI_RES) && K < 2304) ? 2 : 3;
}

cudaError_t tc_gemm_bf16(const bf16 *A, const bf16 *W, int M, int N, int K, int epi,
                         const EpiParams &ep, int max_ctas, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if (K % GBK || N % 64 || max_ctas < 1) return cudaErrorInvalidValue;
  if (reinterpret_cast<uintptr_t>(A) % 16 || reinterpret_cast<uintptr_t>(W) % 16)
    return cudaErrorInvalidValue;
  const int tm = (M + GBM - 1) / GBM;
  const int mc = pair_mode_for(tm, max_ctas, epi, K);
  const GemmPlan g = plan_gemm(M, N, K, max_ctas, mc, ep.ws ? ep.ws_elems : 0);
  switch (g.bn) {
    case 256: return dispatch_mc<256>(A, W, M, N, K, epi, ep, max_ctas, mc, g.ks, s);
    case 192: return dispatch_mc<192>(A, W, M, N, K, epi, ep, max_ctas, mc, g.ks, s);
    case 160: return dispatch_mc<160>(A, W, M, N, K, epi, ep, max_ctas, mc, g.ks, s);
    case 128: return dispatch_mc<128>(A, W, M, N, K, epi, ep, max_ctas, mc, g.ks, s);
    default: return dispatch_mc<64>(A, W, M, N, K, epi, ep, max_ctas, mc, g.ks, s);
  }
}

// Force-load every GEMM kernel instance the dispatch can select (CUDA lazy loading
// would otherwise load a never-launched variant -- e.g. single-CTA tiles chosen
// because the occupancy emulator holds SMs -- on first launch, and loading may
// need a context synchronisation, which never completes while the emulator's
// resident kernel runs: a deadlock observed on B200 with the C2 shapes).
namespace {
template <int BN, int MC>
void preload_bn_mc(cudaFuncAttributes *a) {
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_STORE, MC, 0>);
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_GELU, MC, 0>);
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_GATED_RES, MC, 0>);
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_RES, MC, 0>);
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_QKV, MC, 0>);
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_F32, MC, 0>);
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_CONV, MC, 0>);
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_GEGLU, MC, 0>);
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_CONV, MC, 1>);
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_F32, MC, 1>);
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_CONV, MC, 2>);
  cudaFuncGetAttributes(a, tc_gemm_kernel<BN, EPI_F32, MC, 2>);
}
template <int BN>
void preload_bn(cudaFuncAttributes *a) {
  preload_bn_mc<BN, 1>(a);
  preload_bn_mc<BN, 2>(a);
  preload_bn_mc<BN, 3>(a);
}
}  // namespace

cudaError_t tc_gemm_preload() {
  cudaFuncAttributes a;
  preload_bn<256>(&a);
  preload_bn<192>(&a);
  preload_bn<160>(&a);
  preload_bn<128>(&a);
  preload_bn<64>(&a);
  cudaFuncGetAttributes(&a, splitk_reduce_kernel<EPI_STORE>);
  cudaFuncGetAttributes(&a, splitk_reduce_kernel<EPI_GELU>);
  cudaFuncGetAttributes(&a, splitk_reduce_kernel<EPI_GATED_RES>);
  cudaFuncGetAttributes(&a, splitk_reduce_kernel<EPI_RES>);
  cudaFuncGetAttributes(&a, splitk_reduce_kernel<EPI_QKV>);
  cudaFuncGetAttributes(&a, splitk_reduce_kernel<EPI_F32>);
  cudaFuncGetAttributes(&a, splitk_reduce_kernel<EPI_CONV>);
  cudaFuncGetAttributes(&a, splitk_reduce_kernel<EPI_GEGLU>);
  return cudaGetLastError();
}

// Implicit-GEMM 3x3 conv: out = epi(conv(P) . W^T) with P the halo-padded input
// [h+2, W+2, B, C] and W [N, 9C] (column (ky*3 + kx)*C + c); mode 0 stride 1, mode 1
// stride 2 (output (oy, ox) reads padded rows / columns 2 oy + ky, 2 ox + kx: a 4-D
// tensor map with element strides 2 over the pixel and row dimensions).
bool tc_conv_implicit_ok(int h, int W, int B, int C, int N, int mode) {
  if (C % GBK || N % 64 || (mode != 0 && mode != 1)) return false;
  if (mode == 1 && (h % 2 || W % 2)) return false;
  const int wb = (mode == 1 ? W / 2 : W) * B;
  return wb > 0 && (wb % GBM == 0 || GBM % wb == 0);
}
cudaError_t tc_conv3x3_bf16(const bf16 *P, const bf16 *Wt, int h, int W, int B, int C, int N,
                            int epi, const EpiParams &ep, int max_ctas, cudaStream_t s, int mode) {
  if (h <= 0) return cudaSuccess;
  if (!tc_conv_implicit_ok(h, W, B, C, N, mode) || max_ctas < 1) return cudaErrorInvalidValue;
  const ConvGeo g{W, B, C};
  const int M = mode == 1 ? h / 2 * (W / 2) * B : h * W * B, tm = (M + GBM - 1) / GBM;
  const int mc = pair_mode_for(tm, max_ctas, epi, 9 * C);
  const GemmPlan gp = plan_gemm(M, N, 9 * C, max_ctas, mc, ep.ws ? ep.ws_elems : 0);
  const int ks = gp.ks;
#define STADI_CONV_CASE(BNV)                                                          \
  case BNV:                                                                           \
    return mc == 3   ? dispatch_conv<BNV, 3>(P, Wt, h, g, N, epi, ep, max_ctas, ks, mode, s) \
           : mc == 2 ? dispatch_conv<BNV, 2>(P, Wt, h, g, N, epi, ep, max_ctas, ks, mode, s) \
                     : dispatch_conv<BNV, 1>(P, Wt, h, g, N, epi, ep, max_ctas, ks, mode, s);
  switch (gp.bn) {
    STADI_CONV_CASE(256)
    STADI_CONV_CASE(192)
    STADI_CONV_CASE(160)
    STADI_CONV_CASE(128)
    STADI_CONV_CASE(64)
  }
  return cudaErrorInvalidValue;
#undef STADI_CONV_CASE
}

}  // namespace stadi
