// Kernel-level C entry points (include/stadi_kernels.h).
#include "../../include/stadi_kernels.h"
#include <algorithm>

#include "common.h"
#include "kernels.h"

using namespace stadi;

namespace {
stadi_status cu(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return STADI_OK;
  if (e == cudaErrorInvalidValue)
    return fail(nullptr, STADI_EINVAL, "%s: unsupported shape / argument", what);
  return fail(nullptr, STADI_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}
}  // namespace

namespace {
int device_sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}
EpiParams to_epi(const stadi_k_epi *e) {
  EpiParams ep{};
  ep.bias = e->bias;
  ep.out = e->out;
  ep.ldo = e->ldo;
  ep.res = e->res;
  ep.ldr = e->ldr;
  ep.gate = e->gate;
  ep.gate_bstride = e->gate_bstride;
  ep.B = e->B > 0 ? e->B : 1;
  ep.q = e->q;
  ep.kv_a = e->kv_a;
  ep.kv_b = e->kv_b;
  ep.kv_row0 = e->kv_row0;
  ep.d = e->d;
  ep.ws = e->ws;
  ep.ws_elems = e->ws ? e->ws_elems : 0;
  return ep;
}
}  // namespace

extern "C" stadi_status stadi_k_gemm(int32_t dtype, const void *A, const void *W, int32_t M,
                                     int32_t N, int32_t K, int32_t epi, const stadi_k_epi *e,
                                     void *stream) {
  return stadi_k_gemm_ex(dtype, A, W, M, N, K, epi, e, 0, stream);
}

extern "C" stadi_status stadi_k_gemm_ex(int32_t dtype, const void *A, const void *W, int32_t M,
                                        int32_t N, int32_t K, int32_t epi, const stadi_k_epi *e,
                                        int32_t max_ctas, void *stream) {
  if (!A || !W || !e || M < 0 || N <= 0 || K <= 0 || epi < 0 || epi > 7 || max_ctas < 0 ||
      (e->gate && (e->gate_bstride & 1)) || (e->res && (e->ldr & 1)))
    return fail(nullptr, STADI_EINVAL, "stadi_k_gemm: bad argument");
  const EpiParams ep = to_epi(e);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == STADI_DTYPE_BF16) {
    const int sms = device_sm_count();
    const int ctas = max_ctas ? std::min<int>(max_ctas, sms) : sms;
    return cu(tc_gemm_bf16((const bf16 *)A, (const bf16 *)W, M, N, K, epi, ep, ctas, s),
              "tc_gemm_bf16");
  }
  if (dtype == STADI_DTYPE_FP32_DEBUG)
    return cu(simt_gemm<float>((const float *)A, (const float *)W, M, N, K, epi, ep, s),
              "simt_gemm");
  return fail(nullptr, STADI_EINVAL, "stadi_k_gemm: bad dtype");
}

extern "C" stadi_status stadi_k_attention(int32_t dtype, const void *q, const void *kv, void *o,
                                          int32_t Nq, int32_t Nkv, int32_t B, int32_t H,
                                          int32_t hd, void *stream) {
  if (!q || !kv || !o || Nq < 0 || Nkv <= 0 || B <= 0 || H <= 0 || hd <= 0)
    return fail(nullptr, STADI_EINVAL, "stadi_k_attention: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == STADI_DTYPE_BF16)
    return cu(tc_attention_bf16((const bf16 *)q, (const bf16 *)kv, (bf16 *)o, Nq, Nkv, B, H, hd,
                                s),
              "tc_attention_bf16");
  if (dtype == STADI_DTYPE_FP32_DEBUG)
    return cu(simt_attention<float>((const float *)q, (const float *)kv, (float *)o, Nq, Nkv, B,
                                    H, hd, s),
              "simt_attention");
  return fail(nullptr, STADI_EINVAL, "stadi_k_attention: bad dtype");
}

extern "C" stadi_status stadi_k_ln_modulate(int32_t dtype, const float *x, void *y, int32_t M,
                                            int32_t d, int32_t B, const float *shift,
                                            const float *scale, int32_t bstride, void *stream) {
  if (!x || !y || !shift || !scale || M < 0 || d <= 0 || B <= 0)
    return fail(nullptr, STADI_EINVAL, "stadi_k_ln_modulate: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == STADI_DTYPE_BF16)
    return cu(ln_modulate<bf16>(x, (bf16 *)y, M, d, B, shift, scale, bstride, 1, s), "ln_modulate");
  return cu(ln_modulate<float>(x, (float *)y, M, d, B, shift, scale, bstride, 1, s),
            "ln_modulate");
}

extern "C" uint64_t stadi_k_launch_count(void) { return g_launches; }

extern "C" stadi_status stadi_k_groupnorm(int32_t dtype, const float *x, int32_t h, int32_t W,
                                          int32_t B, int32_t C, const float *gamma,
                                          const float *beta, float eps, int32_t act, int32_t pad,
                                          double *stats, double *ws, uint32_t *ticket, void *out,
                                          void *stream) {
  if (!x || !gamma || !beta || !stats || !ws || !ticket || !out || h < 0 || W <= 0 || B <= 0 ||
      B > 2 || C <= 0 || C % 32 || C > 3072)
    return fail(nullptr, STADI_EINVAL, "stadi_k_groupnorm: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  const stadi_status sp = cu(gn_partials(x, (long)h * W * B, B, C, stats, ws, ticket, s),
                             "gn_partials");
  if (sp != STADI_OK) return sp;
  const double n_total = (double)h * W * (C / 32);
  if (dtype == STADI_DTYPE_BF16)
    return cu(gn_apply<bf16>(x, h, W, B, C, stats, 1, n_total, gamma, beta, eps, act, pad,
                             (bf16 *)out, s), "gn_apply");
  return cu(gn_apply<float>(x, h, W, B, C, stats, 1, n_total, gamma, beta, eps, act, pad,
                            (float *)out, s), "gn_apply");
}

extern "C" stadi_status stadi_k_conv3x3(int32_t dtype, const void *P, const void *Wt, int32_t h,
                                        int32_t W, int32_t B, int32_t C, int32_t N, int32_t mode,
                                        int32_t implicit, const float *bias, float *out,
                                        void *stream) {
  stadi_k_epi e{};
  e.bias = bias;
  e.out = out;
  e.ldo = N;
  return stadi_k_conv3x3_ex(dtype, P, Wt, h, W, B, C, N, mode, implicit, &e, 0, stream);
}

extern "C" stadi_status stadi_k_conv3x3_ex(int32_t dtype, const void *P, const void *Wt,
                                           int32_t h, int32_t W, int32_t B, int32_t C, int32_t N,
                                           int32_t mode, int32_t implicit, const stadi_k_epi *ke,
                                           int32_t max_ctas, void *stream) {
  if (!P || !Wt || !ke || !ke->out || h <= 0 || W <= 0 || B <= 0 || C <= 0 || N <= 0 ||
      mode < 0 || mode > 2 || ke->ldo < N || (ke->res && ke->ldr < N) || max_ctas < 0 ||
      (ke->ldo | ke->ldr | ke->gate_bstride) & 1)
    return fail(nullptr, STADI_EINVAL, "stadi_k_conv3x3: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int ho = mode == 1 ? h / 2 : (mode == 2 ? 2 * h : h);
  const int wo = mode == 1 ? W / 2 : (mode == 2 ? 2 * W : W);
  const int M = ho * wo * B, kp = (9 * C + 63) / 64 * 64;
  EpiParams ep{};
  ep.B = B;
  ep.bias = ke->bias;
  ep.out = ke->out;
  ep.ldo = ke->ldo;
  ep.res = ke->res;
  ep.ldr = ke->ldr;
  ep.gate = ke->gate;
  ep.gate_bstride = ke->gate_bstride;
  const int sms = max_ctas ? std::min(max_ctas, device_sm_count()) : device_sm_count();
  // split-K workspace (used when the conv's tiles fill at most half the SMs)
  float *ws = nullptr;
  if (dtype == STADI_DTYPE_BF16 && ke->ws) {  // caller's workspace
    ep.ws = ke->ws;
    ep.ws_elems = ke->ws_elems;
  } else if (dtype == STADI_DTYPE_BF16) {
    ep.ws_elems = (long)M * N * 16;
    cudaError_t e = cudaMallocAsync(&ws, (size_t)ep.ws_elems * 4, s);
    if (e != cudaSuccess) return cu(e, "cudaMallocAsync");
    ep.ws = ws;
  }
  if (dtype == STADI_DTYPE_BF16 && implicit) {
    // mode 2: nearest-x2 upsample into a padded buffer, then the stride-1 implicit conv
    const int hc = mode == 2 ? 2 * h : h, Wc = mode == 2 ? 2 * W : W, mc = mode == 2 ? 0 : mode;
    if (!tc_conv_implicit_ok(hc, Wc, B, C, N, mc)) {
      if (ws) cudaFreeAsync(ws, s);
      return fail(nullptr, STADI_EINVAL, "implicit conv: unsupported geometry");
    }
    const bf16 *src = (const bf16 *)P;
    bf16 *U = nullptr;
    cudaError_t e = cudaSuccess;
    if (mode == 2) {
      e = cudaMallocAsync(&U, (size_t)(hc + 2) * (Wc + 2) * B * C * 2, s);
      if (e == cudaSuccess) e = upsample_pad<bf16>((const bf16 *)P, h, W, B, C, U, s);
      src = U;
    }
    if (e == cudaSuccess)
      e = tc_conv3x3_bf16(src, (const bf16 *)Wt, hc, Wc, B, C, N, EPI_CONV, ep, sms, s, mc);
    if (U) cudaFreeAsync(U, s);
    if (ws) cudaFreeAsync(ws, s);
    return cu(e, "tc_conv3x3_bf16");
  }
  const size_t esz = dtype == STADI_DTYPE_BF16 ? 2 : 4;
  void *A = nullptr;
  cudaError_t e = cudaMallocAsync(&A, (size_t)M * kp * esz, s);
  if (e != cudaSuccess) {
    if (ws) cudaFreeAsync(ws, s);
    return cu(e, "cudaMallocAsync");
  }
  if (dtype == STADI_DTYPE_BF16) {
    e = im2col<bf16>((const bf16 *)P, h, W, B, C, mode, kp, (bf16 *)A, s);
    if (e == cudaSuccess) e = tc_gemm_bf16((const bf16 *)A, (const bf16 *)Wt, M, N, kp, EPI_CONV,
                                           ep, sms, s);
  } else {
    e = im2col<float>((const float *)P, h, W, B, C, mode, kp, (float *)A, s);
    if (e == cudaSuccess) e = simt_gemm<float>((const float *)A, (const float *)Wt, M, N, kp,
                                               EPI_CONV, ep, s);
  }
  cudaFreeAsync(A, s);
  if (ws) cudaFreeAsync(ws, s);
  return cu(e, "conv3x3");
}


extern "C" stadi_status stadi_k_sampler(float *x, const float *eps_raw, int32_t rows, int32_t W,
                                        int32_t C, int32_t p, int32_t c_out, int32_t ld,
                                        int32_t B, float guidance, float A, float Bc, float Cz,
                                        uint64_t seed, uint32_t m, int32_t row0, void *stream) {
  if (!x || !eps_raw || rows < 0 || W <= 0 || C <= 0 || p <= 0 || rows % p || W % p ||
      c_out < C || ld < p * p * c_out || (B != 1 && B != 2) || row0 < 0)
    return fail(nullptr, STADI_EINVAL, "stadi_k_sampler: bad argument");
  return cu(sampler_update(x, eps_raw, rows, W, C, p, c_out, ld, B, guidance, A, Bc, Cz, seed, nullptr,
                           m, row0, (cudaStream_t)stream),
            "sampler_update");
}

extern "C" stadi_status stadi_k_ddpm_noise(float *out, int64_t n, uint64_t seed, uint32_t m,
                                           int64_t e0, void *stream) {
  if (!out || n < 0 || e0 < 0) return fail(nullptr, STADI_EINVAL, "stadi_k_ddpm_noise: bad argument");
  return cu(philox_normal_fill(out, (long)n, seed, m, (long)e0, (cudaStream_t)stream),
            "philox_normal_fill");
}
