// tcgen05 flash attention for sm_100a: a rank's own queries against the
// full-image K/V assembled in an exchange slot (own rows fresh, other ranks'
// rows stale) — SURVEY §2.6 K3, PAPER.md L80/L171 (DistriFusion-style patch
// parallelism with stale activations); also the cross-attention to the text
// tokens.
//
// One CTA = NQT (1 or 2) query tiles of 128 rows of one (head h, batch b).
// Warp roles (FA4-style ping-pong):
//   warp 0        TMA: the Q tiles once; K and V tiles of 128 keys into a
//                 multi-stage ring.  The head dim is split into chunks of
//                 64 (128B swizzle), 32 (64B) and 16 (32B) columns; TMA
//                 zero-fills hd..hd_pad and rows past Nq / Nkv.
//   warp 1        MMA issuer (one thread): S_g = Q_g K_j^T (SS form, M128 x
//                 N128) into TMEM, then O_g += P_g V_j with P_g read from TMEM
//                 (TS form; P overwrites the first 64 columns of S_g as packed
//                 bf16).  Order per key tile j: PV_0(j), S_0(j+1), PV_1(j),
//                 S_1(j+1) — while softmax group 0 works on S_0(j+1) the
//                 tensor core runs PV_1(j) and S_1(j+1), and vice versa.
//   warps 2..    softmax group g (warps 2+4g .. 5+4g; warp w owns TMEM lanes
//                 32 (w % 4) .. +31, so each group covers all 128; one query row per thread = TMEM
//                 lane): S row -> registers (all loads in flight, one wait),
//                 row max, LAZY rescale (O and l are rescaled in TMEM only
//                 when the running max grows by more than 2^8; otherwise the
//                 stale max is kept — exact, the same max scales P, l and O),
//                 P = 2^(s*scale - m) packed to bf16 into TMEM, row sum in fp32.
//                 Epilogue: O / l -> bf16 global.
// O accumulates in TMEM across all key tiles: no per-tile correction pass.
#include <cuda.h>

#include <cstdlib>

#include "../kernels.h"

namespace stadi {

#ifdef STADI_ATTN_TRACE
// Timeline instrumentation (standalone experiments only): clock64 stamps of
// CTA (0,0,0), slot = (event * 2 + group) * 64 + key tile (tiles < 64).
__device__ long long g_attn_trace[16 * 2 * 64];
#define ATTN_TRACE(ev, g, j)                                                           \
  do {                                                                                 \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64)             \
      g_attn_trace[((ev) * 2 + (g)) * 64 + (j)] = clock64();                           \
  } while (0)
#else
#define ATTN_TRACE(ev, g, j) \
  do {                       \
  } while (0)
#endif

bool make_tmap(CUtensorMap *m, const void *base, int rank, const uint64_t *dims,
               const uint64_t *strides_bytes, const uint32_t *box, CUtensorMapSwizzle swz,
               const uint32_t *estr = nullptr);

namespace {

constexpr int AQ = 128;   // query rows per tile
constexpr int AK = 128;   // keys per tile
constexpr float RESCALE_THRESHOLD = 8.f;  // log2 units: keep a stale max up to 2^8

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Blackwell 3-input max (FMNMX3) and packed fp32x2 FMA / add (FFMA2 / FADD2)
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ uint64_t pack_f32x2(float a, float b) {
  uint64_t u;
  asm("mov.b64 %0, {%1, %2};" : "=l"(u) : "f"(a), "f"(b));
  return u;
}
__device__ __forceinline__ void unpack_f32x2(uint64_t u, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(u));
}
__device__ __forceinline__ uint64_t ffma_f32x2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t add_f32x2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// 2^x for a pair on the FMA / ALU pipes instead of MUFU (FA4's trick to relieve
// the 16 op/clk/SM exp unit): n = rint(x) via the 1.5 * 2^23 magic add,
// f = x - n in [-0.5, 0.5], 2^f by a degree-3 fit (max rel. err 7.5e-5, far
// below the bf16 rounding of P), 2^n added into the exponent field.  x is
// clamped at -125 (2^-125 instead of 0: negligible against a row sum >= 1).
__device__ __forceinline__ void ex2_poly_x2(uint64_t xx, float &p0, float &p1) {
  float x0, x1;
  unpack_f32x2(xx, x0, x1);
  xx = pack_f32x2(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
  const float MAGIC = 12582912.f;
  const uint64_t t = add_f32x2(xx, pack_f32x2(MAGIC, MAGIC));
  const uint64_t nf = add_f32x2(t, pack_f32x2(-MAGIC, -MAGIC));
  const uint64_t f = ffma_f32x2(nf, pack_f32x2(-1.f, -1.f), xx);
  uint64_t q = ffma_f32x2(f, pack_f32x2(0.05517161168f, 0.05517161168f),
                          pack_f32x2(0.24261117048f, 0.24261117048f));
  q = ffma_f32x2(q, f, pack_f32x2(0.69326100063f, 0.69326100063f));
  q = ffma_f32x2(q, f, pack_f32x2(0.99992807098f, 0.99992807098f));
  float q0, q1, t0, t1;
  unpack_f32x2(q, q0, q1);
  unpack_f32x2(t, t0, t1);
  p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
  p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}
// Of every 8 column pairs, POLY (a kernel template parameter) use the
// polynomial exp2, the rest MUFU ex2.

// Head-dim chunking: N64 chunks of 64, then N32 of 32, then N16 of 16.
// AKTO != 0: P aliased over S (no separate P region), AKTO keys per tile.  Measured
// on the C5 shape (round 2, hd 72, P over S): 112 keys 774, 144 710, 160 744, 176 529
// TFLOP/s (register spills at 96 registers / 18 warps, fewer ring stages) against 814
// for the separate-P default -- no instance is built; kept for such A/Bs.
template <int N64, int N32, int N16, int NQT_, int AKTO = 0>
struct AttnCfg {
  static constexpr int NQT = NQT_;
  static constexpr bool PALIAS = AKTO != 0;
  static constexpr int HDP = 64 * N64 + 32 * N32 + 16 * N16;
  static constexpr int NCH = N64 + N32 + N16;
  // keys per tile: 112 with two query tiles so that S (2 x 112), O (2 x 80) and a
  // separate P region (2 x 64) fit the 512 TMEM columns; 128 with one tile
  // DUAL: one query tile per CTA and two CTAs per SM (each its own MMA issuer,
  // softmax group and barriers; 256 TMEM columns each) for hd <= 80 -- used for
  // the short-K/V cross-attention, where per-CTA latency, not K/V streaming, rules
  static constexpr bool DUAL = NQT == 1 && 64 * N64 + 32 * N32 + 16 * N16 <= 80;
  static constexpr int MINB = DUAL ? 2 : 1;      // CTAs per SM
  static constexpr uint32_t TMEM_COLS = DUAL ? 256 : 512;
  static constexpr int AKT = AKTO ? AKTO : ((NQT == 2 || DUAL) ? 112 : 128);
  static constexpr int QTILE = AQ * HDP * 2;   // one Q tile (128 rows), bytes
  static constexpr int KTILE = AKT * HDP * 2;  // one K or V tile, bytes
  __host__ __device__ static constexpr int cw(int c) {  // chunk width
    return c < N64 ? 64 : (c < N64 + N32 ? 32 : 16);
  }
  __host__ __device__ static constexpr int ccol(int c) {  // first head-dim column
    return c < N64 ? 64 * c
                   : (c < N64 + N32 ? 64 * N64 + 32 * (c - N64)
                                    : 64 * N64 + 32 * N32 + 16 * (c - N64 - N32));
  }
  // all chunks 16 wide (32B swizzle): the V tile is one MN-major operand of N = HDP
  // (16-column atoms AKT * 32 bytes apart), so PV is ONE MMA per 16 keys
  static constexpr bool NARROW = N64 == 0 && N32 == 0;
  __host__ __device__ static constexpr int qoff(int c) { return AQ * ccol(c) * 2; }
  __host__ __device__ static constexpr int koff(int c) { return AKT * ccol(c) * 2; }
  __host__ __device__ static constexpr uint32_t cswz(int c) {
    return cw(c) == 64 ? SWZ_128B : (cw(c) == 32 ? SWZ_64B : SWZ_32B);
  }
#ifndef STADI_ATTN_SMEM_KB
#define STADI_ATTN_SMEM_KB 200
#endif
#ifndef STADI_ATTN_MAX_STAGES
#define STADI_ATTN_MAX_STAGES 4
#endif
  static constexpr int STAGES_FIT =
      ((DUAL ? 100 : (PALIAS ? 224 : STADI_ATTN_SMEM_KB)) * 1024 - NQT * QTILE) / (2 * KTILE);
  static constexpr int STAGES =
      STAGES_FIT > STADI_ATTN_MAX_STAGES ? STADI_ATTN_MAX_STAGES : STAGES_FIT;
  static constexpr int OFF_K = NQT * QTILE;
  static constexpr int OFF_V = OFF_K + STAGES * KTILE;
  static constexpr int OFF_BAR = OFF_V + STAGES * KTILE;
  // SPLIT threads share a query row: half 0 owns key columns [0, 64), half 1
  // [64, AKT); they exchange partial row maxima / sums through RED
  // [2 parities][2 groups][SPLIT][128]
  static constexpr int SPLIT = 2;
  static constexpr int W0 = 64, W1 = AKT - 64;
  static constexpr int OFF_RED = OFF_BAR + 512;
  static constexpr int RED_BYTES = 2 * 2 * SPLIT * 128 * 4;
  static constexpr int SMEM = OFF_RED + RED_BYTES + 1024;
  static constexpr int THREADS = 64 + 128 * SPLIT * NQT;
  // TMEM columns: S_g, then O_g (HDP wide), then P_g (packed bf16, AKT / 2 <= 64)
  __host__ __device__ static constexpr uint32_t s_col(int g) { return (uint32_t)(AKT * g); }
  __host__ __device__ static constexpr uint32_t o_col(int g) {
    return (uint32_t)(NQT * AKT + HDP * g);
  }
  __host__ __device__ static constexpr uint32_t p_col(int g) {
    return (uint32_t)(NQT * (AKT + HDP) + 64 * g);
  }
  static_assert(NQT * (AKT + HDP + (PALIAS ? 0 : 64)) <= (int)TMEM_COLS, "TMEM columns");
  static_assert(AKT % 16 == 0 && AKT <= 256, "key tile");
  static_assert(!DUAL || 2 * (SMEM + 1024) <= 228 * 1024, "two CTAs per SM");
  static_assert(NQT == 1 || HDP <= 80, "two query tiles need HDP <= 80");
  static_assert(STAGES >= 2, "smem");
  static_assert(SMEM <= 227 * 1024, "smem");
  static_assert(W1 % 16 == 0 && W1 > 0, "column split");
};

// Load columns [c0, c0 + 16 * n) of this lane's TMEM row into v (fp32).
template <int N>
__device__ __forceinline__ void tmem_row_load(uint32_t taddr, float *v) {
  static_assert(N % 16 == 0, "");
  uint32_t *r = reinterpret_cast<uint32_t *>(v);
#pragma unroll
  for (int c = 0; c + 32 <= N; c += 32) tmem_ld32_nowait(taddr + c, r + c);
  if constexpr (N % 32) tmem_ld16_nowait(taddr + (N - 16), r + (N - 16));
  tmem_ld_wait();
}
template <int N>
__device__ __forceinline__ void tmem_row_store(uint32_t taddr, const float *v) {
  const uint32_t *r = reinterpret_cast<const uint32_t *>(v);
#pragma unroll
  for (int c = 0; c + 32 <= N; c += 32) tmem_st32(taddr + c, r + c);
  if constexpr (N % 32) tmem_st16(taddr + (N - 16), r + (N - 16));
}

// Softmax of one key tile for the W key columns [colb, colb + W) of this
// thread's query row: returns the tile's partial row sum and stores P (bf16
// pairs) into TMEM at p_addr.  v holds the S values (already loaded).
template <int W, int POLY>
__device__ __forceinline__ float softmax_tile(float *v, uint64_t sc2, uint64_t nm2,
                                              uint32_t *pk) {
  uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
  for (int c = 0; c < W; c += 2) {
    const uint64_t xx = ffma_f32x2(pack_f32x2(v[c], v[c + 1]), sc2, nm2);
    float p0, p1;
    if ((c / 2) % 8 < POLY) {
      ex2_poly_x2(xx, p0, p1);
    } else {
      float x0, x1;
      unpack_f32x2(xx, x0, x1);
      p0 = ex2(x0);
      p1 = ex2(x1);
    }
    acc[(c / 2) & 3] = add_f32x2(acc[(c / 2) & 3], pack_f32x2(p0, p1));
    __nv_bfloat162 t2 = __floats2bfloat162_rn(p0, p1);
    pk[c / 2] = *reinterpret_cast<uint32_t *>(&t2);
  }
  const uint64_t t = add_f32x2(add_f32x2(acc[0], acc[1]), add_f32x2(acc[2], acc[3]));
  float r0, r1;
  unpack_f32x2(t, r0, r1);
  return r0 + r1;
}
template <int W>
__device__ __forceinline__ void tmem_load_cols(uint32_t taddr, float *v) {
  uint32_t *r = reinterpret_cast<uint32_t *>(v);
#pragma unroll
  for (int c = 0; c + 32 <= W; c += 32) tmem_ld32_nowait(taddr + c, r + c);
  if constexpr (W % 32) tmem_ld16_nowait(taddr + (W - 16), r + (W - 16));
  tmem_ld_wait();
}
template <int NP>  // NP packed columns (multiple of 8)
__device__ __forceinline__ void tmem_store_packed(uint32_t taddr, const uint32_t *pk) {
#pragma unroll
  for (int c = 0; c + 16 <= NP; c += 16) tmem_st16(taddr + c, pk + c);
  if constexpr (NP % 16) tmem_st8(taddr + (NP - 8), pk + (NP - 8));
}

template <int N64, int N32, int N16, int NQT, int POLY, int QUAD, int AKTO = 0>
__global__ void __launch_bounds__(AttnCfg<N64, N32, N16, NQT, AKTO>::THREADS,
                                  AttnCfg<N64, N32, N16, NQT, AKTO>::MINB)
    tc_attn_kernel(const __grid_constant__ CUtensorMap tq64, const __grid_constant__ CUtensorMap tq32,
                   const __grid_constant__ CUtensorMap tq16, const __grid_constant__ CUtensorMap tk64,
                   const __grid_constant__ CUtensorMap tk32, const __grid_constant__ CUtensorMap tk16,
                   bf16 *__restrict__ out, int Nq, int Nkv, int B, int H, int hd, float scale_log2,
                   int flags) {  // bit 0: exp-phase tokens, bit 1: deferred PV wait (QUAD), bit 2: MMA order
  using C = AttnCfg<N64, N32, N16, NQT, AKTO>;
  constexpr int AKT = C::AKT;
  constexpr bool WM = C::HDP <= 48;  // warp-collective MMA issue (see the MMA issuer)
  // QUAD == 2: P aliased over S.  PV_g(j) and S_g(j+1) are issued back to back once
  // P_g(j) is stored and committed to ONE barrier (s_full), so a key tile costs each
  // group two handoffs (s_full, p_full) instead of four: s_full(j) also tells the group
  // that PV_g(j-1) is done (O may be rescaled, the S/P columns rewritten).
  constexpr bool ALIAS = QUAD == 2 && NQT == 2;
  // P stored over S: the alias MMA order above, or (AKTO, single-tile K/V <= AKT only:
  // the launcher guarantees n_kv == 1, so no S(j+1) can overwrite an unread P)
  constexpr bool POS = ALIAS || C::PALIAS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sQ = smem;
  uint8_t *sK = smem + C::OFF_K;
  uint8_t *sV = smem + C::OFF_V;
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
  uint64_t *q_full = bar;
  uint64_t *k_full = bar + 1, *k_empty = k_full + C::STAGES;
  uint64_t *v_full = k_empty + C::STAGES, *v_empty = v_full + C::STAGES;
  uint64_t *s_full = v_empty + C::STAGES;  // [2] S_g(j) computed
  uint64_t *s_free = s_full + 2;           // [2] S_g(j) read by the softmax group
  uint64_t *p_full = s_free + 2;           // [2] P_g(j) stored
  uint64_t *o_done = p_full + 2;           // [2] PV_g(j) complete (P_g free, O_g final)
  uint64_t *tok = o_done + 2;              // [2] exp-phase tokens (groups alternate)
  uint64_t *tok4 = tok + 2;                // [2][4] per-SMSP exp-phase tokens (QUAD)
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tok4 + 8);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q0 = blockIdx.x * (AQ * NQT), h = blockIdx.y, b = blockIdx.z;
  const int n_kv = (Nkv + AKT - 1) / AKT;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&s_full[g], 1);
      // QUAD: one elected arrival per softmax warp (8 per group); else per thread
      constexpr int ARR = QUAD ? 4 * C::SPLIT : 128 * C::SPLIT;
      mbar_init(&s_free[g], ARR);
      mbar_init(&p_full[g], ARR);
      mbar_init(&o_done[g], 1);
      mbar_init(&tok[g], ARR);
      for (int k = 0; k < 4; ++k) mbar_init(&tok4[g * 4 + k], 2);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // Q / K / V written by the predecessor (QKV GEMM) are complete

  // TMA of one tile of every head-dim chunk (row: first token coordinate)
  auto load_tile = [&](const CUtensorMap *m64, const CUtensorMap *m32, const CUtensorMap *m16,
                       uint8_t *dst, uint64_t *br, int zb, int row, int rows) {
#pragma unroll
    for (int c = 0; c < C::NCH; ++c) {
      const CUtensorMap *m = C::cw(c) == 64 ? m64 : (C::cw(c) == 32 ? m32 : m16);
      tma_load_4d(m, dst + rows * C::ccol(c) * 2, br, C::ccol(c), h, zb, row);
    }
  };

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------ TMA producer
      if (N64) tma_prefetch(&tq64), tma_prefetch(&tk64);
      if (N32) tma_prefetch(&tq32), tma_prefetch(&tk32);
      if (N16) tma_prefetch(&tq16), tma_prefetch(&tk16);
      mbar_expect_tx(q_full, NQT * C::QTILE);
#pragma unroll
      for (int g = 0; g < NQT; ++g)
        load_tile(&tq64, &tq32, &tq16, sQ + g * C::QTILE, q_full, b, q0 + g * AQ, AQ);
      int s = 0;
      uint32_t ph = 0;
      for (int j = 0; j < n_kv; ++j) {
        mbar_wait(&k_empty[s], ph ^ 1);
        mbar_expect_tx(&k_full[s], C::KTILE);
        load_tile(&tk64, &tk32, &tk16, sK + s * C::KTILE, &k_full[s], 2 * b, j * AKT, AKT);
        mbar_wait(&v_empty[s], ph ^ 1);
        mbar_expect_tx(&v_full[s], C::KTILE);
        load_tile(&tk64, &tk32, &tk16, sV + s * C::KTILE, &v_full[s], 2 * b + 1, j * AKT, AKT);
        if (++s == C::STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (WM || lane == 0) {  // ------------------------------------- MMA issuer
      constexpr uint32_t id_s = umma_idesc_bf16(128, AKT, 0, 0);
      // WM (HDP <= 48): descriptors built once before the key loop and advanced by
      // 16-byte offsets, issued by the whole warp (one lane elected in the asm) -- many
      // small N <= 32 MMAs, issue-bound.  Otherwise one thread issues with per-chunk
      // descriptors: measured faster for hd 64 / 72 (814 vs 753 TFLOP/s at C5), where
      // back-to-back issue of the N = 112 S MMAs slows the softmax groups' TMEM traffic.
      uint64_t qdesc[C::NQT][C::NCH], kdesc[C::NCH];
      if constexpr (WM) {
#pragma unroll
        for (int c = 0; c < C::NCH; ++c) {
          const uint32_t sbo = 8 * C::cw(c) * 2;
#pragma unroll
          for (int g = 0; g < C::NQT; ++g)
            qdesc[g][c] = umma_desc(smem_u32(sQ + g * C::QTILE) + C::qoff(c), 16, sbo, C::cswz(c));
          kdesc[c] = umma_desc(smem_u32(sK) + C::koff(c), 16, sbo, C::cswz(c));
        }
      }
      auto issue_s = [&](int g, int st) {
#ifdef STADI_ATTN_NOSMMA  // timing experiment only (wrong results): no S MMAs
        if (st >= 0) return;
#endif
        const uint32_t dt = tmem + C::s_col(g);
        if constexpr (WM) {
          const uint64_t so = (uint64_t)((uint32_t)st * (uint32_t)(C::KTILE >> 4));
          int kk = 0;
#pragma unroll
          for (int c = 0; c < C::NCH; ++c) {
#pragma unroll
            for (int k = 0; k < C::cw(c) / 16; ++k, ++kk)
              umma_bf16_w(dt, qdesc[g][c] + (uint64_t)(2 * k), kdesc[c] + so + (uint64_t)(2 * k),
                          id_s, kk != 0);
          }
        } else {
          const uint32_t qa = smem_u32(sQ + g * C::QTILE), ka = smem_u32(sK + st * C::KTILE);
          int kk = 0;
#pragma unroll
          for (int c = 0; c < C::NCH; ++c) {
            const uint32_t sbo = 8 * C::cw(c) * 2;
            const uint64_t qd0 = umma_desc(qa + C::qoff(c), 16, sbo, C::cswz(c));
            const uint64_t kd0 = umma_desc(ka + C::koff(c), 16, sbo, C::cswz(c));
#pragma unroll
            for (int k = 0; k < C::cw(c) / 16; ++k, ++kk)
              umma_bf16(dt, qd0 + (uint64_t)(2 * k), kd0 + (uint64_t)(2 * k), id_s, kk != 0);
          }
        }
      };
      auto issue_pv = [&](int g, int st, int j) {
#ifdef STADI_ATTN_NOPV  // timing experiment only (wrong results): no PV MMAs
        if (st >= 0) return;
#endif
        // P: AKT / 2 columns of packed bf16 (its own region, or over S when ALIAS)
        const uint32_t pa = tmem + (POS ? C::s_col(g) : C::p_col(g));
        const uint32_t va = smem_u32(sV + st * C::KTILE);
        if constexpr (C::NARROW) {
          constexpr uint32_t idp = umma_idesc_bf16(128, C::HDP, 0, 1);
          const uint32_t dt = tmem + C::o_col(g);
          const uint64_t vd0 = umma_desc(va, AKT * 32, 8 * 32, SWZ_32B);
#pragma unroll
          for (int k = 0; k < AKT / 16; ++k) {  // 16 keys x 32 B = 512 B = 32 units per step
            if constexpr (WM) umma_bf16_ts_w(dt, pa + k * 8, vd0 + (uint64_t)(32 * k), idp, (j | k) != 0);
            else umma_bf16_ts(dt, pa + k * 8, vd0 + (uint64_t)(32 * k), idp, (j | k) != 0);
          }
        } else {
#pragma unroll
          for (int c = 0; c < C::NCH; ++c) {
            const uint32_t rb = C::cw(c) * 2;
            const uint32_t idp = umma_idesc_bf16(128, C::cw(c), 0, 1);
            const uint32_t dt = tmem + C::o_col(g) + C::ccol(c);
            const uint64_t vd0 = umma_desc(va + C::koff(c), AKT * rb, 8 * rb, C::cswz(c));
#pragma unroll
            for (int k = 0; k < AKT / 16; ++k) {
              if constexpr (WM) umma_bf16_ts_w(dt, pa + k * 8, vd0 + (uint64_t)(k * rb), idp, (j | k) != 0);
              else umma_bf16_ts(dt, pa + k * 8, vd0 + (uint64_t)(k * rb), idp, (j | k) != 0);
            }
          }
        }
      };
      auto mma_commit = [&](uint64_t *bar) {
        if constexpr (WM) umma_commit_w(bar);
        else umma_commit(bar);
      };
      // Order per key tile j: S_g(j+1) as soon as the group has read S_g(j) (it
      // overlaps that group's exp work), then PV_g(j) once P_g(j) is stored.
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
#pragma unroll
      for (int g = 0; g < NQT; ++g) {
        issue_s(g, 0);
        mma_commit(&s_full[g]);
      }
      mma_commit(&k_empty[0]);
      int ks = 1 % C::STAGES, vs = 0;
      uint32_t kph = (ks == 0), vph = 0;
      if constexpr (ALIAS) {
        // per tile j and group g: wait P_g(j), PV_g(j), S_g(j+1) into the same
        // columns (in-order tensor pipe: PV reads P before S overwrites it), one commit
        for (int j = 0; j < n_kv; ++j) {
          mbar_wait(&v_full[vs], vph);
          const bool more = j + 1 < n_kv;
          if (more) mbar_wait(&k_full[ks], kph);
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            mbar_wait(&p_full[g], j & 1);
            ATTN_TRACE(2, g, j);
            tc_fence_after();
            issue_pv(g, vs, j);
            if (more) issue_s(g, ks);
            mma_commit(&s_full[g]);
            ATTN_TRACE(8, g, j);
          }
          mma_commit(&v_empty[vs]);
          if (++vs == C::STAGES) {
            vs = 0;
            vph ^= 1;
          }
          if (more) {
            mma_commit(&k_empty[ks]);
            if (++ks == C::STAGES) {
              ks = 0;
              kph ^= 1;
            }
          }
        }
      } else if (NQT == 2 && (flags & 4)) {
        // Event order S_0(j+1), PV_1(j-1), S_1(j+1), PV_0(j): each S is issued as
        // soon as its group has read the previous S, not queued behind the other
        // group's PV of the same tile (which waits for that group's whole exp phase).
        int pvs = 0;  // V slot of tile j-1
        for (int j = 0; j < n_kv; ++j) {
          if (j + 1 < n_kv) {
            mbar_wait(&k_full[ks], kph);
            mbar_wait(&s_free[0], j & 1);
            ATTN_TRACE(0, 0, j);
            tc_fence_after();
            issue_s(0, ks);
            mma_commit(&s_full[0]);
            ATTN_TRACE(1, 0, j);
          }
          if (j > 0) {
            mbar_wait(&p_full[1], (j - 1) & 1);
            ATTN_TRACE(2, 1, j - 1);
            tc_fence_after();
            issue_pv(1, pvs, j - 1);
            mma_commit(&o_done[1]);
            mma_commit(&v_empty[pvs]);
            ATTN_TRACE(8, 1, j - 1);
          }
          if (j + 1 < n_kv) {
            mbar_wait(&s_free[1], j & 1);
            ATTN_TRACE(0, 1, j);
            tc_fence_after();
            issue_s(1, ks);
            mma_commit(&s_full[1]);
            mma_commit(&k_empty[ks]);
            ATTN_TRACE(1, 1, j);
            if (++ks == C::STAGES) {
              ks = 0;
              kph ^= 1;
            }
          }
          mbar_wait(&v_full[vs], vph);
          mbar_wait(&p_full[0], j & 1);
          ATTN_TRACE(2, 0, j);
          tc_fence_after();
          issue_pv(0, vs, j);
          mma_commit(&o_done[0]);
          ATTN_TRACE(8, 0, j);
          pvs = vs;
          if (++vs == C::STAGES) {
            vs = 0;
            vph ^= 1;
          }
        }
        mbar_wait(&p_full[1], (n_kv - 1) & 1);
        tc_fence_after();
        issue_pv(1, pvs, n_kv - 1);
        mma_commit(&o_done[1]);
        mma_commit(&v_empty[pvs]);
      } else {
      for (int j = 0; j < n_kv; ++j) {
        ATTN_TRACE(13, 0, j);
        if (j + 1 < n_kv) {
          mbar_wait(&k_full[ks], kph);
          ATTN_TRACE(14, 0, j);
#pragma unroll
          for (int g = 0; g < NQT; ++g) {
            mbar_wait(&s_free[g], j & 1);
            ATTN_TRACE(0, g, j);
            tc_fence_after();
            issue_s(g, ks);
            mma_commit(&s_full[g]);
            ATTN_TRACE(1, g, j);
          }
          mma_commit(&k_empty[ks]);
          if (++ks == C::STAGES) {
            ks = 0;
            kph ^= 1;
          }
        }
        ATTN_TRACE(13, 1, j);
        mbar_wait(&v_full[vs], vph);
        ATTN_TRACE(14, 1, j);
#pragma unroll
        for (int g = 0; g < NQT; ++g) {
          mbar_wait(&p_full[g], j & 1);
          ATTN_TRACE(2, g, j);
          tc_fence_after();
          issue_pv(g, vs, j);
          mma_commit(&o_done[g]);
          ATTN_TRACE(8, g, j);
        }
        mma_commit(&v_empty[vs]);
        if (++vs == C::STAGES) {
          vs = 0;
          vph ^= 1;
        }
      }
      }
    }
  } else if constexpr (QUAD) {  // ------------------------------ softmax groups (quad rows)
    // warp w >= 2: group g = (w - 2) / 8; TMEM lane quarter w % 4, of which the
    // warp takes the 16-lane half hf.  16x256b TMEM shape: the four threads of
    // a quad share query rows r0 = lb + lane / 4 and r0 + 8 and split every
    // 8-key block by column pairs (2 (lane % 4), +1), so the row max / sum is two
    // shuffles — no shared-memory exchange, no named barrier — and the bf16 P
    // pair of a thread is one 16x128b column (key pair / 2) it owns.
    constexpr int NR = AKT / 8;      // 8-key repetitions per S tile
    constexpr int NO = C::HDP / 8;   // 8-column repetitions of O
    const int sw = warp - 2;
    const int g = sw / 8, hf = (sw % 8) / 4;
    const int qd = warp & 3;
    const int lb = qd * 32 + hf * 16;
    const int cq = 2 * (lane & 3);
    const uint32_t lane_off = (uint32_t)lb << 16;
    const uint32_t s_addr = tmem + lane_off + C::s_col(g);
    const uint32_t p_addr = tmem + lane_off + (POS ? C::s_col(g) : C::p_col(g));
    const uint32_t o_addr = tmem + lane_off + C::o_col(g);
    float m_run[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(&s_full[g], j & 1);
      if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(3, g, j);
      tc_fence_after();
      const int valid = Nkv - j * AKT;
      float v[4 * NR];
#ifdef STADI_ATTN_NOSLOAD  // timing experiment only (wrong results): no S read
#pragma unroll
      for (int i = 0; i < 4 * NR; ++i) v[i] = (float)(i + j) * 1e-3f;
#else
      tmem_ld_q256<NR>(s_addr, reinterpret_cast<uint32_t *>(v));
      tmem_ld_wait();
#endif
      if constexpr (!ALIAS) {  // ALIAS: S is rewritten only after P_g(j) -- no s_free
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[g]);
      }
      if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(4, g, j);
      if (valid < AKT) {
#pragma unroll
        for (int i = 0; i < 4 * NR; ++i)
          if (8 * (i / 4) + cq + (i & 1) >= valid) v[i] = -INFINITY;
      }
      uint64_t acc[2][2];
      uint32_t pk[2 * NR];
      // P = 2^(s scale - m_run) for this thread's pairs, partial row sums in acc; with
      // `track` also the tile's row maxima of the raw scores (am, per row rr)
      auto exp_pass = [&](bool track, float *am) {
        const uint64_t sc2 = pack_f32x2(scale_log2, scale_log2);
        const uint64_t nm2[2] = {pack_f32x2(-m_run[0], -m_run[0]),
                                 pack_f32x2(-m_run[1], -m_run[1])};
        acc[0][0] = acc[0][1] = acc[1][0] = acc[1][1] = 0;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            if (track) am[rr] = fmax3(am[rr], v[4 * r + 2 * rr], v[4 * r + 2 * rr + 1]);
            const uint64_t xx =
                ffma_f32x2(pack_f32x2(v[4 * r + 2 * rr], v[4 * r + 2 * rr + 1]), sc2, nm2[rr]);
            float p0, p1;
#ifdef STADI_ATTN_NOEXP  // timing experiment only (wrong results): no exp work
            if (true) {
              unpack_f32x2(xx, p0, p1);
            } else
#endif
            if (r % 8 < POLY) {
              ex2_poly_x2(xx, p0, p1);
            } else {
              float x0, x1;
              unpack_f32x2(xx, x0, x1);
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            acc[rr][r & 1] = add_f32x2(acc[rr][r & 1], pack_f32x2(p0, p1));
            __nv_bfloat162 t2 = __floats2bfloat162_rn(p0, p1);
            pk[2 * r + rr] = *reinterpret_cast<uint32_t *>(&t2);
          }
        }
      };
      auto rescale_o = [&](const float *factor) {
        static_assert(NO % 2 == 0, "O rescale in 16-column pieces");
#pragma unroll
        for (int c = 0; c < NO; c += 2) {  // 16 columns at a time: S values stay live
          float o[8];
          tmem_ld_q256_x2(o_addr + 8 * c, reinterpret_cast<uint32_t *>(o));
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 8; ++i) o[i] *= factor[(i >> 1) & 1];
          tmem_st_q256_x2(o_addr + 8 * c, reinterpret_cast<const uint32_t *>(o));
        }
      };
      auto token_wait = [&] {
        // exp-phase tokens: the two groups take turns on the exp units, per group
        // (bit 0) or per SM sub-partition (bit 3: the two warps of each group that
        // share an SMSP's MUFU hand over to the other group's two warps there)
        if (NQT == 2 && (flags & 8)) {
          if (g == 1) mbar_wait(&tok4[4 + (warp & 3)], j & 1);
          else if (j > 0) mbar_wait(&tok4[warp & 3], (j - 1) & 1);
        } else if (NQT == 2 && (flags & 1)) {
          if (g == 1) mbar_wait(&tok[1], j & 1);
          else if (j > 0) mbar_wait(&tok[0], (j - 1) & 1);
        }
      };
      bool wait_now = false;
      {
        float mt[2];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          float a0 = -INFINITY, a1 = -INFINITY;  // two independent FMNMX3 chains
#pragma unroll
          for (int r = 0; r < NR; r += 2) {
            a0 = fmax3(a0, v[4 * r + 2 * rr], v[4 * r + 2 * rr + 1]);
            if (r + 1 < NR) a1 = fmax3(a1, v[4 * r + 4 + 2 * rr], v[4 * r + 4 + 2 * rr + 1]);
          }
          float m = fmaxf(a0, a1);
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
          m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
          mt[rr] = m * scale_log2;
        }
        if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(5, g, j);
        float factor[2] = {1.f, 1.f};
        bool grow = false;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          if (mt[rr] > m_run[rr] + RESCALE_THRESHOLD) {
            factor[rr] = ex2(m_run[rr] - mt[rr]);  // 0 on the first tile
            m_run[rr] = mt[rr];
            grow = true;
          }
        }
        // PV_g(j-1) must be complete before O is rescaled or P_g overwritten.  With
        // `defer` the wait moves to just before the P store unless this warp rescales,
        // so the PV latency overlaps the token wait and the exp phase.
        const bool any_grow = __any_sync(0xffffffffu, grow);
        // ALIAS: s_full(j) already implied PV_g(j-1) complete
        wait_now = !ALIAS && j > 0 && (!(flags & 2) || any_grow);
        if (wait_now) {
          mbar_wait(&o_done[g], (j - 1) & 1);
          tc_fence_after();
        }
        if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(9, g, j);
        if (j > 0 && any_grow) rescale_o(factor);
        l[0] *= factor[0];
        l[1] *= factor[1];
        token_wait();
        if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(7, g, j);
        exp_pass(false, nullptr);
      }
      if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(10, g, j);
      if (!ALIAS && j > 0 && !wait_now) {
        mbar_wait(&o_done[g], (j - 1) & 1);
        tc_fence_after();
      }
      if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(11, g, j);
#ifndef STADI_ATTN_NOPST  // timing experiment only (wrong results): no P store
      tmem_st_q128<NR>(p_addr, pk);
#else
      if (pk[0] == 0x12345u) tmem_st_q128<NR>(p_addr, pk);
#endif
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        float s0, s1, s2, s3;
        unpack_f32x2(acc[rr][0], s0, s1);
        unpack_f32x2(acc[rr][1], s2, s3);
        l[rr] += (s0 + s1) + (s2 + s3);
      }
      if (NQT == 2 && (flags & 8)) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&tok4[(1 - g) * 4 + (warp & 3)]);
      } else if (NQT == 2 && (flags & 1)) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&tok[1 - g]);
      }
      tmem_st_wait();
      if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(12, g, j);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[g]);
      if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(6, g, j);
    }
    // epilogue: quad-reduce the row sums, O / l -> bf16 (rows past Nq are padding)
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      l[rr] += __shfl_xor_sync(0xffffffffu, l[rr], 1);
      l[rr] += __shfl_xor_sync(0xffffffffu, l[rr], 2);
    }
    if constexpr (ALIAS) mbar_wait(&s_full[g], n_kv & 1);  // the commit after PV_g(n-1)
    else mbar_wait(&o_done[g], (n_kv - 1) & 1);
    tc_fence_after();
    float o[4 * NO];
    tmem_ld_q256<NO>(o_addr, reinterpret_cast<uint32_t *>(o));
    tmem_ld_wait();
    const int d = H * hd;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int qrow = q0 + g * AQ + lb + (lane >> 2) + 8 * rr;
      if (qrow >= Nq) continue;
      const float inv = 1.f / l[rr];
      bf16 *dst = out + ((long)qrow * B + b) * d + h * hd;
#pragma unroll
      for (int r = 0; r < NO; ++r) {
        const int c = 8 * r + cq;
        if (c < hd)
          *reinterpret_cast<__nv_bfloat162 *>(dst + c) =
              __floats2bfloat162_rn(o[4 * r + 2 * rr] * inv, o[4 * r + 2 * rr + 1] * inv);
      }
    }
  } else {  // ------------------------------------------------------ softmax groups
    // warp w >= 2: group g, column half hf; TMEM lane quarter w % 4 (each group's
    // 8 warps cover all 128 rows twice)
    constexpr int SPLIT = C::SPLIT;
    const int sw = warp - 2;
    const int g = sw / (4 * SPLIT), hf = (sw % (4 * SPLIT)) / 4;
    const int qd = warp & 3;
    const int r = qd * 32 + lane;  // query row within the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const uint32_t st_addr = tmem + lane_off + C::s_col(g) + hf * C::W0;
    const uint32_t p_addr = tmem + lane_off + C::p_col(g) + hf * (C::W0 / 2);
    const uint32_t o_addr = tmem + lane_off + C::o_col(g);
    const int colb = hf * C::W0;  // first key column of this thread
    float *red = reinterpret_cast<float *>(smem + C::OFF_RED);
    auto red_at = [&](int par, int half) -> float & {
      return red[((par * 2 + g) * SPLIT + half) * 128 + r];
    };
    auto group_sync = [&] {
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(128 * SPLIT) : "memory");
    };
    float m_run = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(&s_full[g], j & 1);
      if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(3, g, j);
      tc_fence_after();
      const int valid = Nkv - j * AKT;  // columns >= valid are padding (last tile only)
      float v[C::W0];                   // W1 <= W0
      if (hf == 0) tmem_load_cols<C::W0>(st_addr, v);
      else tmem_load_cols<C::W1>(st_addr, v);
      tc_fence_before();
      mbar_arrive(&s_free[g]);  // S_g may be overwritten by S_g(j+1)
      if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(4, g, j);
      const int W = hf == 0 ? C::W0 : C::W1;
      if (valid < AKT) {
#pragma unroll
        for (int c = 0; c < C::W0; ++c)
          if (c >= W || colb + c >= valid) v[c] = -INFINITY;
      } else if (hf == 1) {
#pragma unroll
        for (int c = C::W1; c < C::W0; ++c) v[c] = -INFINITY;
      }
      // row max: four independent FMNMX3 chains, then the pair's
      float a0 = -INFINITY, a1 = -INFINITY, a2 = -INFINITY, a3 = -INFINITY;
#pragma unroll
      for (int c = 0; c < C::W0; c += 8) {
        a0 = fmax3(a0, v[c], v[c + 1]);
        a1 = fmax3(a1, v[c + 2], v[c + 3]);
        a2 = fmax3(a2, v[c + 4], v[c + 5]);
        a3 = fmax3(a3, v[c + 6], v[c + 7]);
      }
      float mt = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
      red_at(j & 1, hf) = mt;
      group_sync();
      mt = fmaxf(red_at(j & 1, 0), red_at(j & 1, 1)) * scale_log2;
      if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(5, g, j);
      // lazy rescale: move the reference max only when it grows by > 2^8
      float factor = 1.f;
      const bool grow = mt > m_run + RESCALE_THRESHOLD;
      if (grow) {
        factor = ex2(m_run - mt);  // 0 on the first tile (m_run = -inf)
        m_run = mt;
      }
      // P_g and O_g are in use by PV_g(j-1) until o_done completes its j-th phase
      if (j > 0) {
        mbar_wait(&o_done[g], (j - 1) & 1);
        tc_fence_after();
      }
      if (j > 0 && __any_sync(0xffffffffu, grow)) {
#pragma unroll
        for (int c = 0; c < C::HDP; c += 16) {  // the pair rescales alternate pieces
          if ((c / 16) % SPLIT != hf) continue;
          float o[16];
          tmem_row_load<16>(o_addr + c, o);
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] *= factor;
          tmem_row_store<16>(o_addr + c, o);
        }
      }
      l *= factor;
      // exp phase: the two groups take turns (the SM's 16 ex2/clk are shared), so
      // one group's S read / max exchange overlaps the other group's exps
      if constexpr (NQT == 2) {
        if (g == 1) mbar_wait(&tok[1], j & 1);
        else if (j > 0) mbar_wait(&tok[0], (j - 1) & 1);
      }
      if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(7, g, j);
      const uint64_t sc2 = pack_f32x2(scale_log2, scale_log2), nm2 = pack_f32x2(-m_run, -m_run);
      uint32_t pk[C::W0 / 2];
      if (hf == 0) {
        l += softmax_tile<C::W0, POLY>(v, sc2, nm2, pk);
        tmem_store_packed<C::W0 / 2>(p_addr, pk);
      } else {
        l += softmax_tile<C::W1, POLY>(v, sc2, nm2, pk);
        tmem_store_packed<C::W1 / 2>(p_addr, pk);
      }
      if constexpr (NQT == 2) mbar_arrive(&tok[1 - g]);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[g]);
      if (hf == 0 && qd == 2 && lane == 0) ATTN_TRACE(6, g, j);
    }
    // epilogue: O / l; the pair combines its partial row sums, then each thread
    // stores its alternate 16-column pieces (rows beyond Nq are padding)
    group_sync();  // every thread is past its last tile's max exchange
    red_at(0, hf) = l;
    group_sync();
    l = red_at(0, 0) + red_at(0, 1);
    mbar_wait(&o_done[g], (n_kv - 1) & 1);
    tc_fence_after();
    const int qrow = q0 + g * AQ + r;
    const float inv = 1.f / l;
    const int d = H * hd;
    bf16 *dst = out + ((long)qrow * B + b) * d + h * hd;
#pragma unroll
    for (int c = 0; c < C::HDP; c += 16) {
      if ((c / 16) % SPLIT != hf) continue;
      float o[16];
      tmem_row_load<16>(o_addr + c, o);
      if (qrow < Nq) {
        if ((hd & 7) == 0) {
#pragma unroll
          for (int e = 0; e < 16; e += 8) {
            if (c + e < hd) {
              __nv_bfloat162 b0 = __floats2bfloat162_rn(o[e] * inv, o[e + 1] * inv);
              __nv_bfloat162 b1 = __floats2bfloat162_rn(o[e + 2] * inv, o[e + 3] * inv);
              __nv_bfloat162 b2 = __floats2bfloat162_rn(o[e + 4] * inv, o[e + 5] * inv);
              __nv_bfloat162 b3 = __floats2bfloat162_rn(o[e + 6] * inv, o[e + 7] * inv);
              *reinterpret_cast<uint4 *>(dst + c + e) =
                  make_uint4(*reinterpret_cast<uint32_t *>(&b0), *reinterpret_cast<uint32_t *>(&b1),
                             *reinterpret_cast<uint32_t *>(&b2), *reinterpret_cast<uint32_t *>(&b3));
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (c + e < hd) dst[c + e] = __float2bfloat16_rn(o[e] * inv);
        }
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

// Run-time switches (A/B measurements, C5 shape 16384 x 16384, hd 72, B200, round 2
// tools/gpu_attn_env.sh): exp-phase tokens per group 787 TFLOP/s, no tokens 807, per-SMSP
// tokens (the two warps of a group on one sub-partition hand the MUFU to the other
// group's two warps there) 816; MMA order S_0(j+1), PV_1(j-1), S_1(j+1), PV_0(j) +1%.
// Defaults: per-SMSP tokens + that MMA order.
// STADI_ATTN_TOK=1: per-group tokens instead (TOK=0 together with TOK4=0: none);
// STADI_ATTN_TOK4=0: no per-SMSP tokens;
// STADI_ATTN_DEFER=0: wait for PV(j-1) before the rescale check, not before the P store;
// STADI_ATTN_ORDER=0: MMA issue order S_0(j+1), S_1(j+1), PV_0(j), PV_1(j).
int attn_flags() {
  static const int v = [] {
    const char *e = getenv("STADI_ATTN_TOK"), *d = getenv("STADI_ATTN_DEFER"),
               *o = getenv("STADI_ATTN_ORDER");
    const char *t4 = getenv("STADI_ATTN_TOK4");
    const bool tok4 = !(t4 && t4[0] == '0');
    return ((e && e[0] == '1') ? 1 : 0) | ((d && d[0] == '0') ? 0 : 2) |
           ((o && o[0] == '0') ? 0 : 4) | (tok4 && !(e && e[0] == '1') ? 8 : 0);
  }();
  return v;
}
template <int N64, int N32, int N16, int NQT, int POLY, int QUAD, int AKTO = 0>
cudaError_t launch_attn_p(const bf16 *q, const bf16 *kv, bf16 *o, int Nq, int Nkv, int B, int H,
                        int hd, cudaStream_t s) {
  using C = AttnCfg<N64, N32, N16, NQT, AKTO>;
  const int d = H * hd;
  if (d % 8) return cudaErrorInvalidValue;  // TMA: 16-byte row strides
  CUtensorMap tm[6] = {};
  const uint64_t dq[4] = {(uint64_t)hd, (uint64_t)H, (uint64_t)B, (uint64_t)Nq};
  const uint64_t sq[3] = {(uint64_t)hd * 2, (uint64_t)d * 2, (uint64_t)B * d * 2};
  const uint64_t dk[4] = {(uint64_t)hd, (uint64_t)H, (uint64_t)2 * B, (uint64_t)Nkv};
  const uint64_t sk[3] = {(uint64_t)hd * 2, (uint64_t)d * 2, (uint64_t)2 * B * d * 2};
  const int widths[3] = {64, 32, 16};
  const int present[3] = {N64, N32, N16};
  const CUtensorMapSwizzle swz[3] = {CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_SWIZZLE_64B,
                                     CU_TENSOR_MAP_SWIZZLE_32B};
  bool ok = true;
  for (int i = 0; i < 3; ++i) {
    if (!present[i]) continue;
    const uint32_t qbox[4] = {(uint32_t)widths[i], 1, 1, (uint32_t)AQ};
    const uint32_t kbox[4] = {(uint32_t)widths[i], 1, 1, (uint32_t)C::AKT};
    ok &= make_tmap(&tm[i], q, 4, dq, sq, qbox, swz[i]);
    ok &= make_tmap(&tm[3 + i], kv, 4, dk, sk, kbox, swz[i]);
  }
  if (!ok) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_attn_kernel<N64, N32, N16, NQT, POLY, QUAD, AKTO>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((Nq + AQ * NQT - 1) / (AQ * NQT), H, B);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)hd);
  cudaError_t el = launch_pdl(tc_attn_kernel<N64, N32, N16, NQT, POLY, QUAD, AKTO>, grid,
                              dim3(C::THREADS), C::SMEM, s, tm[0], tm[1], tm[2], tm[3], tm[4],
                              tm[5], o, Nq, Nkv, B, H, hd, scale_log2, attn_flags());
  if (el != cudaSuccess) return el;
  ++g_launches;
  return cudaGetLastError();
}

// STADI_ATTN_POLY=k (0..4): k of every 8 column pairs take the polynomial exp2
// (default 0: measured on B200 the exp units are not the bound of this kernel);
// for A/B measurements of the MUFU / FMA balance.
int attn_poly() {
  static const int v = [] {
    const char *e = getenv("STADI_ATTN_POLY");
    const int k = e ? atoi(e) : 0;
    return k < 0 ? 0 : (k > 4 ? 4 : k);
  }();
  return v;
}
// STADI_ATTN_QUAD=0 selects the column-split softmax layout (two threads per row in
// different warps, max exchange through shared memory) for A/B measurements.
int attn_quad() {
  static const int v = [] {
    const char *e = getenv("STADI_ATTN_QUAD");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v;
}
// STADI_ATTN_ALIAS=1: P aliased over S, two handoffs per key tile and group instead of
// four (QUAD == 2).  Measured slower on the C5 shape (774 vs 815 TFLOP/s: S(j+1) can no
// longer overlap the group's exp phase), so off by default; it is parity-tested.
int attn_alias() {
  static const int v = [] {
    const char *e = getenv("STADI_ATTN_ALIAS");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return v;
}
// Short K/V (cross-attention, Nkv <= 128) on the two-CTAs-per-SM variant: one 128-key
// tile with P over S (S 128 + O HDP <= 256 TMEM columns) instead of two 112-key tiles
// (the PixArt text has 120 tokens, SD / SDXL 77).  STADI_ATTN_XTILE=0 disables.
int attn_xtile() {
  static const int v = [] {
    const char *e = getenv("STADI_ATTN_XTILE");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v;
}
template <int N64, int N32, int N16, int NQT>
cudaError_t launch_attn(const bf16 *q, const bf16 *kv, bf16 *o, int Nq, int Nkv, int B, int H,
                        int hd, cudaStream_t s) {
  if constexpr (NQT == 1 && 64 * N64 + 32 * N32 + 16 * N16 <= 80) {
    if (Nkv <= 128 && attn_xtile() && attn_quad())
      return launch_attn_p<N64, N32, N16, NQT, 0, 1, 128>(q, kv, o, Nq, Nkv, B, H, hd, s);
  }
  if (!attn_quad()) return launch_attn_p<N64, N32, N16, NQT, 0, 0>(q, kv, o, Nq, Nkv, B, H, hd, s);
  if (NQT == 2 && attn_alias() && attn_poly() == 0)
    return launch_attn_p<N64, N32, N16, NQT, 0, 2>(q, kv, o, Nq, Nkv, B, H, hd, s);
  switch (attn_poly()) {
    case 0: return launch_attn_p<N64, N32, N16, NQT, 0, 1>(q, kv, o, Nq, Nkv, B, H, hd, s);
    case 1: return launch_attn_p<N64, N32, N16, NQT, 1, 1>(q, kv, o, Nq, Nkv, B, H, hd, s);
    case 2: return launch_attn_p<N64, N32, N16, NQT, 2, 1>(q, kv, o, Nq, Nkv, B, H, hd, s);
    case 4: return launch_attn_p<N64, N32, N16, NQT, 4, 1>(q, kv, o, Nq, Nkv, B, H, hd, s);
    default: return launch_attn_p<N64, N32, N16, NQT, 3, 1>(q, kv, o, Nq, Nkv, B, H, hd, s);
  }
}

}  // namespace

// hd 72 / 80: 16-wide (32B-swizzled) head-dim chunks, one PV MMA of N = 80 per 16
// keys (measured 8% faster than 64 + 16 chunks); STADI_ATTN_NARROW=0 switches back.
int attn_narrow() {
  static const int v = [] {
    const char *e = getenv("STADI_ATTN_NARROW");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v;
}

int attn_dual40() {
  static const int v = [] {
    const char *e = getenv("STADI_ATTN_DUAL40");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v;
}

// Force-load every attention kernel instance (see tc_gemm_preload).
namespace {
template <int N64, int N32, int N16, int NQT>
void preload_attn(cudaFuncAttributes *a) {
  cudaFuncGetAttributes(a, tc_attn_kernel<N64, N32, N16, NQT, 0, 0>);
  cudaFuncGetAttributes(a, tc_attn_kernel<N64, N32, N16, NQT, 0, 1>);
  cudaFuncGetAttributes(a, tc_attn_kernel<N64, N32, N16, NQT, 1, 1>);
  cudaFuncGetAttributes(a, tc_attn_kernel<N64, N32, N16, NQT, 2, 1>);
  cudaFuncGetAttributes(a, tc_attn_kernel<N64, N32, N16, NQT, 3, 1>);
  cudaFuncGetAttributes(a, tc_attn_kernel<N64, N32, N16, NQT, 4, 1>);
  cudaFuncGetAttributes(a, tc_attn_kernel<N64, N32, N16, NQT, 0, 2>);
  if constexpr (NQT == 1 && 64 * N64 + 32 * N32 + 16 * N16 <= 80)
    cudaFuncGetAttributes(a, tc_attn_kernel<N64, N32, N16, NQT, 0, 1, 128>);
}
}  // namespace
cudaError_t tc_attention_preload() {
  cudaFuncAttributes a;
  preload_attn<0, 0, 1, 2>(&a);
  preload_attn<0, 1, 1, 2>(&a);
  preload_attn<0, 1, 1, 1>(&a);
  preload_attn<1, 0, 0, 2>(&a);
  preload_attn<0, 0, 5, 2>(&a);
  preload_attn<0, 0, 5, 1>(&a);
  preload_attn<1, 0, 0, 1>(&a);
  preload_attn<1, 0, 1, 2>(&a);
  preload_attn<2, 1, 0, 1>(&a);
  return cudaGetLastError();
}

// K/V lengths up to this use the two-CTAs-per-SM variant (hd 64 / 72 / 80): a few key
// tiles leave each CTA latency bound, so a second resident CTA hides it, and its grid
// of 128-query CTAs fills the SMs twice as finely; for long K/V the shared ping-pong
// CTA wins (786 vs 583 TFLOP/s at 16384 keys).  Measured round 2 (kbench, B200): 1024
// keys hd 80 249 -> 337 TFLOP/s, 1024 keys hd 64 x 20 heads 289 -> 365, 4096 keys hd 64
// 492 -> 603.  STADI_ATTN_DUAL_KV overrides (0 = never).
int attn_dual_max_kv() {
  static const int v = [] {
    const char *e = getenv("STADI_ATTN_DUAL_KV");
    return e ? atoi(e) : 4096;
  }();
  return v;
}

// Supported head dims (padded to hd_pad): 16 (16), 40 (48 = 32 + 16), 64 (64),
// 72 / 80 (80 = 64 + 16), 160 (160 = 64 + 64 + 32, one query tile per CTA).
bool tc_attention_supported(int hd) {
  return hd == 16 || hd == 40 || hd == 64 || hd == 72 || hd == 80 || hd == 160;
}

cudaError_t tc_attention_bf16(const bf16 *q, const bf16 *kv, bf16 *o, int Nq, int Nkv, int B,
                              int H, int hd, cudaStream_t s) {
  if (Nq <= 0) return cudaSuccess;
  if (Nkv <= 0) return cudaErrorInvalidValue;
  switch (hd) {
    case 16: return launch_attn<0, 0, 1, 2>(q, kv, o, Nq, Nkv, B, H, hd, s);
    case 40:  // dual slower for the 77-token cross-attention, faster for 128 < K/V <=
              // STADI_ATTN_DUAL_KV (SD-1.5 level 0, 4096 keys: 329-339 -> 348-371 TFLOP/s);
              // STADI_ATTN_DUAL40=0 keeps the ping-pong CTA
      if (attn_dual40() && Nkv > 128 && Nkv <= attn_dual_max_kv())
        return launch_attn<0, 1, 1, 1>(q, kv, o, Nq, Nkv, B, H, hd, s);
      return launch_attn<0, 1, 1, 2>(q, kv, o, Nq, Nkv, B, H, hd, s);
    case 64:  // dual: SDXL cross-attention 20 -> 16 us
      if (Nkv <= attn_dual_max_kv()) return launch_attn<1, 0, 0, 1>(q, kv, o, Nq, Nkv, B, H, hd, s);
      return launch_attn<1, 0, 0, 2>(q, kv, o, Nq, Nkv, B, H, hd, s);
    case 72:
    case 80:
      if (Nkv <= attn_dual_max_kv())  // cross-attention to the text tokens
        return launch_attn<0, 0, 5, 1>(q, kv, o, Nq, Nkv, B, H, hd, s);
      if (attn_narrow()) return launch_attn<0, 0, 5, 2>(q, kv, o, Nq, Nkv, B, H, hd, s);
      return launch_attn<1, 0, 1, 2>(q, kv, o, Nq, Nkv, B, H, hd, s);
    case 160: return launch_attn<2, 1, 0, 1>(q, kv, o, Nq, Nkv, B, H, hd, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace stadi
