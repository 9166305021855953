// Device helpers for sm_100a: dtype conversion, mbarrier, TMA, tcgen05 PTX.
// Bit layouts of the UMMA shared-memory / instruction descriptors follow the
// PTX ISA tcgen05 "matrix descriptor" and "instruction descriptor" tables.
#pragma once
#include <utility>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace stadi {

using bf16 = __nv_bfloat16;

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.f + tanhf(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float silu(float x) { return x / (1.f + expf(-x)); }
__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.f + erff(x * 0.7071067811865476f));
}

// ----------------------------------------------------------------- GEMM epilogues
// Shared by the SIMT (fp32 debug) and the tcgen05 GEMM so both paths compute
// exactly the same post-accumulation math.
enum EpiKind : int {
  EPI_STORE = 0,      // out[T]   = acc + bias
  EPI_GELU = 1,       // out[T]   = gelu_tanh(acc + bias)
  EPI_GATED_RES = 2,  // res[f32] += gate[row % B] * (acc + bias)   (adaLN gate, DiT ref [4])
  EPI_RES = 3,        // res[f32] += acc + bias
  EPI_QKV = 4,        // cols [0,d): q ; [d,3d): K/V into exchange slot(s)
  EPI_F32 = 5,        // outf[f32] = acc + bias
  EPI_CONV = 6,       // outf[f32] = acc + bias (+ gate[row % B][col]) (+ res[row][col])
  EPI_GEGLU = 7,      // out[T][col/2 + j] = v[2j] * gelu_erf(v[2j+1])  (interleaved a|g)
};

struct EpiParams {
  const float *bias;   // [N] or nullptr
  void *out;           // T or float, row stride ldo
  int ldo;
  float *res;          // residual fp32, row stride ldr
  int ldr;
  const float *gate;   // gate row for batch b at gate + b * gate_bstride
  int gate_bstride;
  int B;               // internal batch (rows are token-major, batch innermost)
  void *q;             // EPI_QKV: q [M, d]
  void *kv_a;          // EPI_QKV: K/V slot base ([N_tok, B, 2, d]); own rows at kv_row0
  void *kv_b;          // optional second slot (publish version), may be nullptr
  long kv_row0;        // first own row of the slot = tok_begin * B
  int d;
  float *ws;           // tcgen05 GEMM split-K workspace (fp32 partial tiles), or nullptr
  long ws_elems;
  int res_prefetch;    // tcgen05 GEMM: L2-prefetch the residual tile before the accumulator wait
  int res_vec4;        // tcgen05 GEMM: 16-byte residual read-modify-write when aligned
  // EPI_QKV, IPC transport: the publish version's own K/V rows are also stored straight
  // into n_kv_peer peers' slots (device array of their slot bases, same layout, mapped
  // with CUDA IPC): the variable-size all-gather fused into the epilogue (P2P stores)
  void *const *kv_peer;
  int n_kv_peer;
};

// Apply the epilogue to `n` consecutive columns col..col+n-1 of one row.
template <typename T, int EPI>
__device__ __forceinline__ void epi_apply(const EpiParams &p, int row, int col, float *v, int n) {
  if (p.bias) {
#pragma unroll 8
    for (int i = 0; i < n; ++i) v[i] += __ldg(p.bias + col + i);
  }
  if constexpr (EPI == EPI_STORE || EPI == EPI_GELU) {
    T *o = reinterpret_cast<T *>(p.out) + (long)row * p.ldo + col;
#pragma unroll 8
    for (int i = 0; i < n; ++i) o[i] = from_f<T>(EPI == EPI_GELU ? gelu_tanh(v[i]) : v[i]);
  } else if constexpr (EPI == EPI_F32) {
    float *o = reinterpret_cast<float *>(p.out) + (long)row * p.ldo + col;
#pragma unroll 8
    for (int i = 0; i < n; ++i) o[i] = v[i];
  } else if constexpr (EPI == EPI_GATED_RES || EPI == EPI_RES) {
    float *r = p.res + (long)row * p.ldr + col;
    if constexpr (EPI == EPI_GATED_RES) {
      const float *g = p.gate + (row % p.B) * p.gate_bstride + col;
#pragma unroll 8
      for (int i = 0; i < n; ++i) r[i] += __ldg(g + i) * v[i];
    } else {
#pragma unroll 8
      for (int i = 0; i < n; ++i) r[i] += v[i];
    }
  } else if constexpr (EPI == EPI_CONV) {
    float *o = reinterpret_cast<float *>(p.out) + (long)row * p.ldo + col;
    const float *g = p.gate ? p.gate + (row % p.B) * p.gate_bstride + col : nullptr;
    const float *r = p.res ? p.res + (long)row * p.ldr + col : nullptr;
#pragma unroll 8
    for (int i = 0; i < n; ++i) {
      float a = v[i];
      if (g) a += __ldg(g + i);
      if (r) a += r[i];
      o[i] = a;
    }
  } else if constexpr (EPI == EPI_GEGLU) {
    // n is even and col even: pairs (a_k, g_k) -> one output column k = col/2 + j
    T *o = reinterpret_cast<T *>(p.out) + (long)row * p.ldo + col / 2;
#pragma unroll 8
    for (int j = 0; j < n / 2; ++j) o[j] = from_f<T>(v[2 * j] * gelu_erf(v[2 * j + 1]));
  } else if constexpr (EPI == EPI_QKV) {
    // n consecutive columns never straddle the q / kv boundary (d % n == 0).
    if (col < p.d) {
      T *o = reinterpret_cast<T *>(p.q) + (long)row * p.d + col;
#pragma unroll 8
      for (int i = 0; i < n; ++i) o[i] = from_f<T>(v[i]);
    } else {
      const long off = (p.kv_row0 + row) * 2L * p.d + (col - p.d);
      T *a = reinterpret_cast<T *>(p.kv_a) + off;
#pragma unroll 8
      for (int i = 0; i < n; ++i) a[i] = from_f<T>(v[i]);
      if (p.kv_b) {
        T *b = reinterpret_cast<T *>(p.kv_b) + off;
#pragma unroll 8
        for (int i = 0; i < n; ++i) b[i] = from_f<T>(v[i]);
      }
      for (int k = 0; k < p.n_kv_peer; ++k) {
        T *b = reinterpret_cast<T *>(p.kv_peer[k]) + off;
#pragma unroll 8
        for (int i = 0; i < n; ++i) b[i] = from_f<T>(v[i]);
      }
    }
  }
}

// ----------------------------------------------------------------- PDL
// Programmatic dependent launch: a hot-path kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start (prologue: barrier
// init, TMEM alloc, descriptor prefetch) while its predecessor's last blocks still
// run; every such kernel calls pdl_wait() before touching global memory, which
// returns once the predecessor has completed and its writes are visible.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();  // STADI_PDL=0 disables (tc_gemm.cu)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ----------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
#ifdef STADI_MBAR_SUSPEND  // A/B: explicit suspend-time hint (ns) for the HW wait
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"((uint32_t)STADI_MBAR_SUSPEND)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}
// Wait for the phase with the given parity to complete.  Watchdog: trap after
// ~10 s so a protocol bug becomes a CUDA error instead of a hung GPU.
#ifdef STADI_MBAR_TEST_WAIT  // A/B: non-suspending test_wait spin instead of try_wait
__device__ __forceinline__ bool mbar_test_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
#define mbar_try_wait mbar_test_wait
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  const uint64_t t0 = globaltimer();
  uint32_t it = 0;
  while (!mbar_try_wait(a, parity)) {
    if ((++it & 0x3FFu) == 0 && globaltimer() - t0 > 10000000000ull) __trap();
  }
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_prefetch(const void *tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(const void *tmap, void *dst, uint64_t *bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(const void *tmap, void *dst, uint64_t *bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(const void *tmap, void *dst, uint64_t *bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// Multicast TMA: the box lands at the same smem offset in every CTA of the
// cluster named by cta_mask and signals each destination's mbarrier (same offset).
__device__ __forceinline__ void tma_load_2d_mc(const void *tmap, void *dst, uint64_t *bar, int c0,
                                               int c1, uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

// ---- CTA pair (tcgen05 cta_group::2): the pair's leader (rank 0) issues the MMA;
// operand loads of both CTAs complete on the leader's mbarrier.  A shared::cta
// address with bit 24 cleared names the same offset in the pair's rank-0 CTA.
__device__ __forceinline__ uint32_t pair_leader_addr(const void *p) {
  return smem_u32(p) & 0xFEFFFFFFu;
}
__device__ __forceinline__ void tma_load_2d_cg2(const void *tmap, void *dst, uint64_t *bar, int c0,
                                                int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(pair_leader_addr(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_cg2(const void *tmap, void *dst, uint64_t *bar, int c0,
                                                int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(pair_leader_addr(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_cg2(const void *tmap, void *dst, uint64_t *bar, int c0,
                                                int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(pair_leader_addr(bar))
      : "memory");
}
// Arrive on the mbarrier at the same offset in cluster CTA `rank`.
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
__device__ __forceinline__ void tmem_alloc_cg2(uint32_t *dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_cg2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// D[tmem of both CTAs] (+)= A[smem, 128 rows per CTA] . B[smem, N/2 rows per CTA]^T
__device__ __forceinline__ void umma_bf16_cg2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Commit the leader's MMAs to the mbarrier at this offset in both CTAs of the pair.
__device__ __forceinline__ void umma_commit_cg2(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"((uint16_t)0x3)
      : "memory");
}

// Warp-collective forms: called by a whole converged warp with warp-uniform operands,
// one lane elected inside the asm issues.  The compiler then keeps descriptors in
// uniform registers and emits no per-instruction elect loop / R2UR moves (the
// single-thread forms cost ~13-20 dependent instructions per MMA on B200).
__device__ __forceinline__ void umma_bf16_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_cg2_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_w(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void umma_commit_cg2_w(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}" ::"r"(smem_u32(bar)), "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void umma_commit_mc_w(uint64_t *bar, uint16_t cta_mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}" ::"r"(smem_u32(bar)), "h"(cta_mask)
      : "memory");
}

// tcgen05 ------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate)
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// Commit to the same-offset mbarrier of every CTA in cta_mask (cluster multicast).
__device__ __forceinline__ void umma_commit_mc(uint64_t *bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// 32 lanes x 16 columns
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Issue-only variants: several loads in flight, one tmem_ld_wait() afterwards.
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t *r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t *r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 32 lanes x 32 / 16 consecutive 32-bit columns from registers; tmem_st_wait() before
// the stored values may be consumed (e.g. by a tcgen05.mma after a thread sync).
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t *r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t *r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t *r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                   taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
               "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// ---- 16-lane shapes (a quad of threads shares a TMEM lane) -------------------
// 16x256b: thread t reads lanes base + t/4 and base + t/4 + 8, 32-bit columns
// 2(t%4), 2(t%4)+1 of every 8-column repetition; registers per repetition:
// [lane0 c, lane0 c+1, lane1 c, lane1 c+1].  16x128b: thread t owns column t%4
// of every 4-column repetition; registers per repetition: [lane0, lane1].
#define STADI_R4(i) "=r"(r[i]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3])
#define STADI_W4(i) "r"(r[i]), "r"(r[i + 1]), "r"(r[i + 2]), "r"(r[i + 3])
__device__ __forceinline__ void tmem_ld_q256_x1(uint32_t a, uint32_t *r) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
               : STADI_R4(0)
               : "r"(a));
}
__device__ __forceinline__ void tmem_ld_q256_x2(uint32_t a, uint32_t *r) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : STADI_R4(0), STADI_R4(4)
               : "r"(a));
}
__device__ __forceinline__ void tmem_ld_q256_x4(uint32_t a, uint32_t *r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : STADI_R4(0), STADI_R4(4), STADI_R4(8), STADI_R4(12)
      : "r"(a));
}
__device__ __forceinline__ void tmem_ld_q256_x8(uint32_t a, uint32_t *r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : STADI_R4(0), STADI_R4(4), STADI_R4(8), STADI_R4(12), STADI_R4(16), STADI_R4(20),
        STADI_R4(24), STADI_R4(28)
      : "r"(a));
}
__device__ __forceinline__ void tmem_st_q256_x1(uint32_t a, const uint32_t *r) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), STADI_W4(0)
               : "memory");
}
__device__ __forceinline__ void tmem_st_q256_x2(uint32_t a, const uint32_t *r) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x2.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a),
               STADI_W4(0), STADI_W4(4)
               : "memory");
}
__device__ __forceinline__ void tmem_st_q256_x4(uint32_t a, const uint32_t *r) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a),
      STADI_W4(0), STADI_W4(4), STADI_W4(8), STADI_W4(12)
      : "memory");
}
__device__ __forceinline__ void tmem_st_q256_x8(uint32_t a, const uint32_t *r) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
      STADI_W4(0), STADI_W4(4), STADI_W4(8), STADI_W4(12), STADI_W4(16), STADI_W4(20),
      STADI_W4(24), STADI_W4(28)
      : "memory");
}
__device__ __forceinline__ void tmem_st_q128_x1(uint32_t a, const uint32_t *r) {
  asm volatile("tcgen05.st.sync.aligned.16x128b.x1.b32 [%0], {%1,%2};" ::"r"(a), "r"(r[0]),
               "r"(r[1])
               : "memory");
}
__device__ __forceinline__ void tmem_st_q128_x2(uint32_t a, const uint32_t *r) {
  asm volatile("tcgen05.st.sync.aligned.16x128b.x2.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), STADI_W4(0)
               : "memory");
}
__device__ __forceinline__ void tmem_st_q128_x4(uint32_t a, const uint32_t *r) {
  asm volatile("tcgen05.st.sync.aligned.16x128b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a),
               STADI_W4(0), STADI_W4(4)
               : "memory");
}
__device__ __forceinline__ void tmem_st_q128_x8(uint32_t a, const uint32_t *r) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x128b.x8.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a),
      STADI_W4(0), STADI_W4(4), STADI_W4(8), STADI_W4(12)
      : "memory");
}
#undef STADI_R4
#undef STADI_W4
// NREP repetitions of 16x256b (8 columns each) starting at column offset of a,
// issued as x8 / x4 / x2 / x1 pieces without waiting (tmem_ld_wait() after).
template <int NREP>
__device__ __forceinline__ void tmem_ld_q256(uint32_t a, uint32_t *r) {
  constexpr int N8 = NREP / 8, R8 = NREP % 8;
#pragma unroll
  for (int i = 0; i < N8; ++i) tmem_ld_q256_x8(a + 64 * i, r + 32 * i);
  int rep = 8 * N8;
  if constexpr (R8 & 4) { tmem_ld_q256_x4(a + 8 * rep, r + 4 * rep); rep += 4; }
  if constexpr (R8 & 2) { tmem_ld_q256_x2(a + 8 * rep, r + 4 * rep); rep += 2; }
  if constexpr (R8 & 1) tmem_ld_q256_x1(a + 8 * rep, r + 4 * rep);
}
template <int NREP>
__device__ __forceinline__ void tmem_st_q256(uint32_t a, const uint32_t *r) {
  constexpr int N8 = NREP / 8, R8 = NREP % 8;
#pragma unroll
  for (int i = 0; i < N8; ++i) tmem_st_q256_x8(a + 64 * i, r + 32 * i);
  int rep = 8 * N8;
  if constexpr (R8 & 4) { tmem_st_q256_x4(a + 8 * rep, r + 4 * rep); rep += 4; }
  if constexpr (R8 & 2) { tmem_st_q256_x2(a + 8 * rep, r + 4 * rep); rep += 2; }
  if constexpr (R8 & 1) tmem_st_q256_x1(a + 8 * rep, r + 4 * rep);
}
// NREP repetitions of 16x128b (4 columns each), 2 registers per repetition.
template <int NREP>
__device__ __forceinline__ void tmem_st_q128(uint32_t a, const uint32_t *r) {
  constexpr int N8 = NREP / 8, R8 = NREP % 8;
#pragma unroll
  for (int i = 0; i < N8; ++i) tmem_st_q128_x8(a + 32 * i, r + 16 * i);
  int rep = 8 * N8;
  if constexpr (R8 & 4) { tmem_st_q128_x4(a + 4 * rep, r + 2 * rep); rep += 4; }
  if constexpr (R8 & 2) { tmem_st_q128_x2(a + 4 * rep, r + 2 * rep); rep += 2; }
  if constexpr (R8 & 1) tmem_st_q128_x1(a + 4 * rep, r + 2 * rep);
}
// D[tmem] (+)= A[tmem] * B[smem], kind::f16: A (K-major, 2 bf16 per 32-bit column,
// lane = row) lives in tensor memory (the "TS" form).
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// UMMA shared-memory matrix descriptor (sm_100): start>>4 [0,14), LBO>>4
// [16,30), SBO>>4 [32,46), version 1 [46,48), base offset 0, swizzle [61,64):
// 0 none, 2 = 128B, 4 = 64B, 6 = 32B.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t swz) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)swz << 61);
}
constexpr uint32_t SWZ_128B = 2, SWZ_64B = 4, SWZ_32B = 6;

// Instruction descriptor kind::f16: D f32, A/B bf16, K-major unless *_mn set.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

}  // namespace stadi
