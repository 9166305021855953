// tcgen05 flash attention for sm_100a: a rank's own queries against the
// full-image K/V assembled in an exchange slot (own rows fresh, other ranks'
// rows stale) — SURVEY §2.6 K3, PAPER.md L80/L171 (DistriFusion-style patch
// parallelism with stale activations).
//
// One CTA = one (128-query tile, head h, batch b).  Warp roles:
//   warp 0      TMA: Q once; K and V tiles of 128 keys into a 3-stage ring
//               (head dim split into a 128B-swizzled 64-wide part and a
//               32B-swizzled 16-wide remainder; TMA zero-fills hd..hd_pad)
//   warp 1      MMA issuer: S_j = Q K_j^T (M=128, N=128, K=hd_pad) into one of
//               two TMEM S buffers; O_j = P_j V_j (M=128, N=hd_pad) into one of
//               two TMEM O buffers (V is the MN-major B operand)
//   warps 2-5   softmax: one query row per thread — running max / sum in
//               fp32 (exp2), P_j as bf16 into 128B-swizzled smem, then the
//               lagged correction O_acc = O_acc * 2^(m_ref - m_j) + O_j in
//               registers, normalise and store.
// S_{j+1} is computed while the softmax warps work on S_j; PV_j overlaps
// softmax_{j+1}.
#include <cuda.h>

#include "../kernels.h"

namespace stadi {

bool make_tmap(CUtensorMap *m, const void *base, int rank, const uint64_t *dims,
               const uint64_t *strides_bytes, const uint32_t *box, CUtensorMapSwizzle swz);

namespace {

constexpr int AQ = 128;   // query rows per CTA
constexpr int AK = 128;   // keys per tile
constexpr int KST = 3;    // K/V pipeline stages

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MAIN, int REM>  // MAIN in {0,64}, REM in {0,16}: hd_pad = MAIN + REM
struct AttnCfg {
  static constexpr int HDP = MAIN + REM;
  static constexpr int MAIN_BYTES = MAIN * 2 * 128;   // 128 rows x MAIN bf16
  static constexpr int REM_BYTES = REM * 2 * 128;
  static constexpr int TILE = MAIN_BYTES + REM_BYTES;  // one Q/K/V tile
  static constexpr int P_BYTES = AQ * AK * 2;          // 32 KB
  // layout: Q | K[KST] | V[KST] | P[2] | barriers
  static constexpr int OFF_K = TILE;
  static constexpr int OFF_V = OFF_K + KST * TILE;
  static constexpr int OFF_P = OFF_V + KST * TILE;
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  // TMEM columns: S buffers at 0 / 128, O buffers at 256 / 384
  __host__ __device__ static constexpr uint32_t s_col(int i) { return i ? 128u : 0u; }
  __host__ __device__ static constexpr uint32_t o_col(int i) { return i ? 384u : 256u; }
};

template <int MAIN, int REM>
__global__ void __launch_bounds__(192, 1)
    tc_attn_kernel(const __grid_constant__ CUtensorMap tq_main,
                   const __grid_constant__ CUtensorMap tq_rem,
                   const __grid_constant__ CUtensorMap tkv_main,
                   const __grid_constant__ CUtensorMap tkv_rem, bf16 *__restrict__ out, int Nq,
                   int Nkv, int B, int H, int hd, float scale_log2) {
  using C = AttnCfg<MAIN, REM>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sQ = smem;
  uint8_t *sK = smem + C::OFF_K;
  uint8_t *sV = smem + C::OFF_V;
  uint8_t *sP = smem + C::OFF_P;
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
  uint64_t *q_full = bar;
  uint64_t *k_full = bar + 1, *k_empty = k_full + KST;
  uint64_t *v_full = k_empty + KST, *v_empty = v_full + KST;
  uint64_t *s_full = v_empty + KST, *p_full = s_full + 2, *o_full = p_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(o_full + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q0 = blockIdx.x * AQ, h = blockIdx.y, b = blockIdx.z;
  const int n_kv = (Nkv + AK - 1) / AK;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_full[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------ TMA producer
      if (MAIN) tma_prefetch(&tq_main), tma_prefetch(&tkv_main);
      if (REM) tma_prefetch(&tq_rem), tma_prefetch(&tkv_rem);
      mbar_expect_tx(q_full, C::TILE);
      if (MAIN) tma_load_4d(&tq_main, sQ, q_full, 0, h, b, q0);
      if (REM) tma_load_4d(&tq_rem, sQ + C::MAIN_BYTES, q_full, MAIN, h, b, q0);
      int s = 0;
      uint32_t ph = 0;
      for (int j = 0; j < n_kv; ++j) {
        mbar_wait(&k_empty[s], ph ^ 1);
        mbar_expect_tx(&k_full[s], C::TILE);
        if (MAIN) tma_load_4d(&tkv_main, sK + s * C::TILE, &k_full[s], 0, h, 2 * b, j * AK);
        if (REM)
          tma_load_4d(&tkv_rem, sK + s * C::TILE + C::MAIN_BYTES, &k_full[s], MAIN, h, 2 * b,
                      j * AK);
        mbar_wait(&v_empty[s], ph ^ 1);
        mbar_expect_tx(&v_full[s], C::TILE);
        if (MAIN) tma_load_4d(&tkv_main, sV + s * C::TILE, &v_full[s], 0, h, 2 * b + 1, j * AK);
        if (REM)
          tma_load_4d(&tkv_rem, sV + s * C::TILE + C::MAIN_BYTES, &v_full[s], MAIN, h, 2 * b + 1,
                      j * AK);
        if (++s == KST) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------ MMA issuer
      constexpr uint32_t id_s = umma_idesc_bf16(128, AK, 0, 0);
      constexpr uint32_t id_pv_main = umma_idesc_bf16(128, MAIN > 0 ? MAIN : 64, 0, 1);
      constexpr uint32_t id_pv_rem = umma_idesc_bf16(128, REM > 0 ? REM : 16, 0, 1);
      const uint32_t q_addr = smem_u32(sQ);
      auto issue_s = [&](int j, int st) {
        const uint32_t dt = tmem + C::s_col(j & 1);
        const uint32_t k_addr = smem_u32(sK + st * C::TILE);
        int kk = 0;
        if (MAIN) {
#pragma unroll
          for (int k = 0; k < MAIN / 16; ++k, ++kk)
            umma_bf16(dt, umma_desc(q_addr + k * 32, 16, 1024, SWZ_128B),
                      umma_desc(k_addr + k * 32, 16, 1024, SWZ_128B), id_s, kk != 0);
        }
        if (REM) {
          umma_bf16(dt, umma_desc(q_addr + C::MAIN_BYTES, 16, 256, SWZ_32B),
                    umma_desc(k_addr + C::MAIN_BYTES, 16, 256, SWZ_32B), id_s, kk != 0);
        }
      };
      mbar_wait(q_full, 0);
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0;
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      issue_s(0, 0);
      umma_commit(&s_full[0]);
      umma_commit(&k_empty[0]);
      ks = 1 % KST;
      kph = (ks == 0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) {
          mbar_wait(&k_full[ks], kph);
          tc_fence_after();
          issue_s(j + 1, ks);
          umma_commit(&s_full[(j + 1) & 1]);
          umma_commit(&k_empty[ks]);
          if (++ks == KST) {
            ks = 0;
            kph ^= 1;
          }
        }
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);
        mbar_wait(&v_full[vs], vph);
        tc_fence_after();
        const uint32_t p_addr = smem_u32(sP + (j & 1) * C::P_BYTES);
        const uint32_t v_addr = smem_u32(sV + vs * C::TILE);
        const uint32_t dt = tmem + C::o_col(j & 1);
#pragma unroll
        for (int k = 0; k < AK / 16; ++k) {
          const uint64_t ad =
              umma_desc(p_addr + (k >> 2) * (AQ * 128) + (k & 3) * 32, 16, 1024, SWZ_128B);
          if (MAIN)
            umma_bf16(dt, ad, umma_desc(v_addr + k * 16 * 128, 128 * 128, 1024, SWZ_128B),
                      id_pv_main, k != 0);
          if (REM)
            umma_bf16(dt + MAIN, ad,
                      umma_desc(v_addr + C::MAIN_BYTES + k * 16 * 32, 128 * 32, 256, SWZ_32B),
                      id_pv_rem, k != 0);
        }
        umma_commit(&o_full[j & 1]);
        umma_commit(&v_empty[vs]);
        if (++vs == KST) {
          vs = 0;
          vph ^= 1;
        }
      }
    }
  } else {  // ------------------------------------------------ softmax warps 2..5
    const int qd = warp & 3;
    const int r = qd * 32 + lane;  // query row within the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    float m = -INFINITY, l = 0.f;
    float m_hist[2] = {0.f, 0.f};
    float m_ref = 0.f;
    float oacc[C::HDP];
#pragma unroll
    for (int c = 0; c < C::HDP; ++c) oacc[c] = 0.f;
    bool have_ref = false;

    auto correction = [&](int i) {
      mbar_wait(&o_full[i & 1], (i >> 1) & 1);
      tc_fence_after();
      const uint32_t ot = tmem + lane_off + C::o_col(i & 1);
      const float mi = m_hist[i & 1];
      const float sc = have_ref ? ex2(m_ref - mi) : 0.f;
      float v[32];
#pragma unroll
      for (int c0 = 0; c0 + 32 <= C::HDP; c0 += 32) {
        tmem_ld32(ot + c0, v);
#pragma unroll
        for (int c = 0; c < 32; ++c) oacc[c0 + c] = oacc[c0 + c] * sc + v[c];
      }
      if constexpr (C::HDP % 32) {
        constexpr int c0 = C::HDP - 16;
        tmem_ld16(ot + c0, v);
#pragma unroll
        for (int c = 0; c < 16; ++c) oacc[c0 + c] = oacc[c0 + c] * sc + v[c];
      }
      m_ref = mi;
      have_ref = true;
      tc_fence_before();
    };

    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t st = tmem + lane_off + C::s_col(j & 1);
      const int valid = Nkv - j * AK;  // columns >= valid are padding
      float v[32];
      float mt = -INFINITY;
#pragma unroll
      for (int c0 = 0; c0 < AK; c0 += 32) {  // pass 1: row max
        tmem_ld32(st + c0, v);
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (c0 + c < valid) mt = fmaxf(mt, v[c]);
      }
      const float m_new = fmaxf(m, mt * scale_log2);
      const float alpha = ex2(m - m_new);  // m = -inf on the first tile -> 0
      float rs = 0.f;
      uint8_t *prow = sP + (j & 1) * C::P_BYTES + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
      for (int c0 = 0; c0 < AK; c0 += 32) {  // pass 2: p = 2^(s - m), bf16 into swizzled smem
        tmem_ld32(st + c0, v);
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          const float p0 = (c0 + c < valid) ? ex2(v[c] * scale_log2 - m_new) : 0.f;
          const float p1 = (c0 + c + 1 < valid) ? ex2(v[c + 1] * scale_log2 - m_new) : 0.f;
          rs += p0 + p1;
          __nv_bfloat162 t2 = __floats2bfloat162_rn(p0, p1);
          pk[c / 2] = *reinterpret_cast<uint32_t *>(&t2);
        }
        const int atom = c0 >> 6;
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // four 16-byte chunks of 8 keys
          const int chunk = ((c0 & 63) >> 3) + u;
          uint4 w = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
          *reinterpret_cast<uint4 *>(prow + atom * (AQ * 128) + ((chunk ^ (r & 7)) << 4)) = w;
        }
      }
      l = l * alpha + rs;
      m = m_new;
      m_hist[j & 1] = m_new;
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&p_full[j & 1]);
      if (j >= 1) correction(j - 1);
    }
    correction(n_kv - 1);
    // normalise + store (rows beyond Nq are padding)
    const int qrow = q0 + r;
    if (qrow < Nq) {
      const float inv = 1.f / l;
      const int d = H * hd;
      bf16 *o = out + ((long)qrow * B + b) * d + h * hd;
#pragma unroll
      for (int c = 0; c < C::HDP; c += 8) {
        if (c < hd) {
          __nv_bfloat162 a0 = __floats2bfloat162_rn(oacc[c] * inv, oacc[c + 1] * inv);
          __nv_bfloat162 a1 = __floats2bfloat162_rn(oacc[c + 2] * inv, oacc[c + 3] * inv);
          __nv_bfloat162 a2 = __floats2bfloat162_rn(oacc[c + 4] * inv, oacc[c + 5] * inv);
          __nv_bfloat162 a3 = __floats2bfloat162_rn(oacc[c + 6] * inv, oacc[c + 7] * inv);
          uint4 w = make_uint4(*reinterpret_cast<uint32_t *>(&a0), *reinterpret_cast<uint32_t *>(&a1),
                               *reinterpret_cast<uint32_t *>(&a2), *reinterpret_cast<uint32_t *>(&a3));
          *reinterpret_cast<uint4 *>(o + c) = w;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int MAIN, int REM>
cudaError_t launch_attn(const bf16 *q, const bf16 *kv, bf16 *o, int Nq, int Nkv, int B, int H,
                        int hd, cudaStream_t s) {
  using C = AttnCfg<MAIN, REM>;
  const int d = H * hd;
  CUtensorMap tq_main{}, tq_rem{}, tkv_main{}, tkv_rem{};
  const uint64_t dq[4] = {(uint64_t)hd, (uint64_t)H, (uint64_t)B, (uint64_t)Nq};
  const uint64_t sq[3] = {(uint64_t)hd * 2, (uint64_t)d * 2, (uint64_t)B * d * 2};
  const uint64_t dk[4] = {(uint64_t)hd, (uint64_t)H, (uint64_t)2 * B, (uint64_t)Nkv};
  const uint64_t sk[3] = {(uint64_t)hd * 2, (uint64_t)d * 2, (uint64_t)2 * B * d * 2};
  const uint32_t bmain[4] = {64, 1, 1, 128}, brem[4] = {16, 1, 1, 128};
  bool ok = true;
  if (MAIN) {
    ok &= make_tmap(&tq_main, q, 4, dq, sq, bmain, CU_TENSOR_MAP_SWIZZLE_128B);
    ok &= make_tmap(&tkv_main, kv, 4, dk, sk, bmain, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  if (REM) {
    ok &= make_tmap(&tq_rem, q, 4, dq, sq, brem, CU_TENSOR_MAP_SWIZZLE_32B);
    ok &= make_tmap(&tkv_rem, kv, 4, dk, sk, brem, CU_TENSOR_MAP_SWIZZLE_32B);
  }
  if (!ok) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_attn_kernel<MAIN, REM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((Nq + AQ - 1) / AQ, H, B);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
  tc_attn_kernel<MAIN, REM><<<grid, 192, C::SMEM, s>>>(tq_main, tq_rem, tkv_main, tkv_rem, o, Nq,
                                                       Nkv, B, H, hd, scale_log2);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace

bool tc_attention_supported(int hd) { return hd == 16 || hd == 64 || hd == 72 || hd == 80; }

cudaError_t tc_attention_bf16(const bf16 *q, const bf16 *kv, bf16 *o, int Nq, int Nkv, int B,
                              int H, int hd, cudaStream_t s) {
  if (Nq <= 0) return cudaSuccess;
  if (Nkv <= 0) return cudaErrorInvalidValue;
  switch (hd) {
    case 16: return launch_attn<0, 16>(q, kv, o, Nq, Nkv, B, H, hd, s);
    case 64: return launch_attn<64, 0>(q, kv, o, Nq, Nkv, B, H, hd, s);
    case 72:
    case 80: return launch_attn<64, 16>(q, kv, o, Nq, Nkv, B, H, hd, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace stadi
