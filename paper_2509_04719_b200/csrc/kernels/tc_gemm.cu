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
//  * warps 2-5: epilogue — tcgen05.ld of the fp32 accumulator (each warp owns
//    its 32-lane TMEM quarter), fused bias / GELU / adaLN-gated residual /
//    K-V-slot scatter, direct global stores;
//  * the accumulator is double-buffered in TMEM (2 x BN columns) so the
//    epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>

#include <mutex>

#include "../kernels.h"

namespace stadi {

namespace {

constexpr int GBM = 128, GBK = 64;

constexpr int EPI_LD = 33;                       // staging row stride (floats, bank-free)
constexpr int EPI_SMEM = 4 * 32 * EPI_LD * 4;    // 4 epilogue warps x 32 x 32 fp32

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = GBM * GBK * 2;              // 16 KB
  static constexpr int B_BYTES = BN * GBK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (196 * 1024) / STAGE > 8 ? 8 : (196 * 1024) / STAGE;
  static constexpr int TMEM_COLS = (2 * BN <= 128) ? 128 : (2 * BN <= 256 ? 256 : 512);
  static constexpr int SMEM = STAGES * STAGE + EPI_SMEM + 1024 /*align*/ + 256 /*barriers*/;
};

// Epilogue of two adjacent columns (col even) of one row, vectorised stores.
template <int EPI>
__device__ __forceinline__ void epi_pair(const EpiParams &p, int row, int col, float v0, float v1) {
  if (p.bias) {
    const float2 b = *reinterpret_cast<const float2 *>(p.bias + col);
    v0 += b.x;
    v1 += b.y;
  }
  if constexpr (EPI == EPI_STORE || EPI == EPI_GELU) {
    if (EPI == EPI_GELU) {
      v0 = gelu_tanh(v0);
      v1 = gelu_tanh(v1);
    }
    *reinterpret_cast<__nv_bfloat162 *>(reinterpret_cast<bf16 *>(p.out) + (long)row * p.ldo +
                                        col) = __floats2bfloat162_rn(v0, v1);
  } else if constexpr (EPI == EPI_F32 || EPI == EPI_CONV) {
    if constexpr (EPI == EPI_CONV) {
      if (p.gate) {
        const float2 g = *reinterpret_cast<const float2 *>(p.gate + (row % p.B) * p.gate_bstride +
                                                           col);
        v0 += g.x;
        v1 += g.y;
      }
      if (p.res) {
        const float2 r = *reinterpret_cast<const float2 *>(p.res + (long)row * p.ldr + col);
        v0 += r.x;
        v1 += r.y;
      }
    }
    *reinterpret_cast<float2 *>(reinterpret_cast<float *>(p.out) + (long)row * p.ldo + col) =
        make_float2(v0, v1);
  } else if constexpr (EPI == EPI_GATED_RES || EPI == EPI_RES) {
    float2 *r = reinterpret_cast<float2 *>(p.res + (long)row * p.ldr + col);
    float2 a = *r;
    if constexpr (EPI == EPI_GATED_RES) {
      const float2 g =
          *reinterpret_cast<const float2 *>(p.gate + (row % p.B) * p.gate_bstride + col);
      a.x += g.x * v0;
      a.y += g.y * v1;
    } else {
      a.x += v0;
      a.y += v1;
    }
    *r = a;
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
    }
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(192, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   int M, int N, int K, EpiParams ep) {
  using C = GemmCfg<BN>;
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
  const int n_tiles = tiles_m * tiles_n;
  const int nkb = K / GBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int mb = tile / tiles_n, nb = tile % tiles_n;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], C::STAGE);
          tma_load_2d(&tmA, sA + s * C::A_BYTES, &full[s], kb * GBK, mb * GBM);
          tma_load_2d(&tmB, sB + s * C::B_BYTES, &full[s], kb * GBK, nb * BN);
          if (++s == C::STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(GBM, BN, 0, 0);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < GBK / 16; ++k) {
            const uint64_t ad = umma_desc(a0 + k * 32, 16, 1024, SWZ_128B);
            const uint64_t bd = umma_desc(b0 + k * 32, 16, 1024, SWZ_128B);
            umma_bf16(dtm, ad, bd, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[s]);
          if (++s == C::STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {  // ---------------------------- epilogue warps 2..5
    const int qd = warp & 3;  // TMEM lane quarter this warp may access
    int it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
      const int mb = tile / tiles_n, nb = tile % tiles_n;
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int row0 = mb * GBM + qd * 32;
      const uint32_t tbase = tmem + ((uint32_t)(qd * 32) << 16) + acc * BN;
      float *stg = stg_all + (warp - 2) * 32 * EPI_LD;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        // TMEM -> registers (lane = row) -> smem, then coalesced: lanes cover
        // 16 column pairs of two rows per step
        float v[32];
        tmem_ld32(tbase + c0, v);
        if (c0 + 32 >= BN) {  // accumulator fully read: release it to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) stg[lane * EPI_LD + i] = v[i];
        __syncwarp();
        const int cc = 2 * (lane & 15);
#pragma unroll 4
        for (int it = 0; it < 16; ++it) {
          const int r = 2 * it + (lane >> 4);
          if (row0 + r < M)
            epi_pair<EPI>(ep, row0 + r, nb * BN + c0 + cc, stg[r * EPI_LD + cc],
                          stg[r * EPI_LD + cc + 1]);
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
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

// Exported for the attention kernel too.
bool make_tmap(CUtensorMap *m, const void *base, int rank, const uint64_t *dims,
               const uint64_t *strides_bytes, const uint32_t *box, CUtensorMapSwizzle swz) {
  EncodeFn fn = get_encode();
  if (!fn) return false;
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = 1;
  }
  for (int i = 0; i < rank - 1; ++i) st[i] = strides_bytes[i];
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void *>(base), d, st, b,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {
template <int BN, int EPI>
cudaError_t launch_gemm(const bf16 *A, const bf16 *W, int M, int N, int K, const EpiParams &ep,
                        int max_ctas, cudaStream_t s) {
  using C = GemmCfg<BN>;
  CUtensorMap ta, tb;
  const uint64_t da[2] = {(uint64_t)K, (uint64_t)M}, sa[1] = {(uint64_t)K * 2};
  const uint32_t ba[2] = {GBK, GBM};
  const uint64_t db[2] = {(uint64_t)K, (uint64_t)N}, sb[1] = {(uint64_t)K * 2};
  const uint32_t bb[2] = {GBK, (uint32_t)BN};
  if (!make_tmap(&ta, A, 2, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_tmap(&tb, W, 2, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  static bool attr_set = false;  // per template instance
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((M + GBM - 1) / GBM) * (N / BN);
  const int grid = tiles < max_ctas ? tiles : max_ctas;
  tc_gemm_kernel<BN, EPI><<<grid, 192, C::SMEM, s>>>(ta, tb, M, N, K, ep);
  ++g_launches;
  return cudaGetLastError();
}

template <int BN>
cudaError_t dispatch_epi(const bf16 *A, const bf16 *W, int M, int N, int K, int epi,
                         const EpiParams &ep, int max_ctas, cudaStream_t s) {
  switch (epi) {
    case EPI_STORE: return launch_gemm<BN, EPI_STORE>(A, W, M, N, K, ep, max_ctas, s);
    case EPI_GELU: return launch_gemm<BN, EPI_GELU>(A, W, M, N, K, ep, max_ctas, s);
    case EPI_GATED_RES: return launch_gemm<BN, EPI_GATED_RES>(A, W, M, N, K, ep, max_ctas, s);
    case EPI_RES: return launch_gemm<BN, EPI_RES>(A, W, M, N, K, ep, max_ctas, s);
    case EPI_QKV: return launch_gemm<BN, EPI_QKV>(A, W, M, N, K, ep, max_ctas, s);
    case EPI_F32: return launch_gemm<BN, EPI_F32>(A, W, M, N, K, ep, max_ctas, s);
    case EPI_CONV: return launch_gemm<BN, EPI_CONV>(A, W, M, N, K, ep, max_ctas, s);
    case EPI_GEGLU: return launch_gemm<BN, EPI_GEGLU>(A, W, M, N, K, ep, max_ctas, s);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t tc_gemm_bf16(const bf16 *A, const bf16 *W, int M, int N, int K, int epi,
                         const EpiParams &ep, int max_ctas, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  if (K % GBK || N % 64 || max_ctas < 1) return cudaErrorInvalidValue;
  if (reinterpret_cast<uintptr_t>(A) % 16 || reinterpret_cast<uintptr_t>(W) % 16)
    return cudaErrorInvalidValue;
  // Pick the N tile that minimises (waves x tile width), preferring wider tiles.
  const int cands[4] = {256, 192, 128, 64};
  int best = 64;
  long best_cost = -1;
  const int tm = (M + GBM - 1) / GBM;
  for (int bn : cands) {
    if (N % bn) continue;
    const long tiles = (long)tm * (N / bn);
    const long waves = (tiles + max_ctas - 1) / max_ctas;
    const long cost = waves * (bn + 32);  // +32: per-tile fixed overhead
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  switch (best) {
    case 256: return dispatch_epi<256>(A, W, M, N, K, epi, ep, max_ctas, s);
    case 192: return dispatch_epi<192>(A, W, M, N, K, epi, ep, max_ctas, s);
    case 128: return dispatch_epi<128>(A, W, M, N, K, epi, ep, max_ctas, s);
    default: return dispatch_epi<64>(A, W, M, N, K, epi, ep, max_ctas, s);
  }
}

}  // namespace stadi
