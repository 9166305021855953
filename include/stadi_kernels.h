/*
 * stadi_kernels.h — kernel-level C entry points of libstadi, for parity tests
 * and micro-benchmarks of the individual hot-path kernels.  All pointers are
 * DEVICE pointers on the current device; all calls are stream-ordered on
 * `stream` (a cudaStream_t, NULL = legacy default stream) and return
 * STADI_EINVAL for unsupported shapes, STADI_ECUDA on a launch error.
 *
 * dtype: STADI_DTYPE_BF16 -> the tcgen05/TMA kernels (bf16 operands, fp32
 * accumulation); STADI_DTYPE_FP32_DEBUG -> the SIMT fp32 kernels.
 */
#ifndef STADI_KERNELS_H_
#define STADI_KERNELS_H_

#include "stadi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* GEMM epilogues, applied to acc = A[M,K] . W[N,K]^T:     */
enum {
  STADI_EPI_STORE = 0,      /* out[T] (ld ldo) = acc + bias                       */
  STADI_EPI_GELU = 1,       /* out[T] = gelu_tanh(acc + bias)                     */
  STADI_EPI_GATED_RES = 2,  /* res[f32] += gate[row % B][col] * (acc + bias)      */
  STADI_EPI_RES = 3,        /* res[f32] += acc + bias                             */
  STADI_EPI_QKV = 4,        /* cols < d: q[T]; cols >= d: K/V rows of the exchange
                               slot(s) kv_a / kv_b at row kv_row0 + row            */
  STADI_EPI_F32 = 5,        /* out[f32] = acc + bias                              */
  STADI_EPI_CONV = 6,       /* out[f32] = acc + bias (+ gate[row % B][col]: the per-
                               batch time-embedding term) (+ res[row][col])      */
  STADI_EPI_GEGLU = 7       /* W rows interleaved (a_0, g_0, a_1, g_1, ...):
                               out[T][row][k] = a_k * gelu_erf(g_k), N/2 columns  */
};

typedef struct {
  const float *bias;   /* [N] or NULL                                          */
  void *out;           /* output (T or f32), row stride ldo elements           */
  int32_t ldo;
  float *res;          /* residual (f32), row stride ldr                       */
  int32_t ldr;
  const float *gate;   /* gate row of batch b at gate + b * gate_bstride        */
  int32_t gate_bstride;
  int32_t B;           /* internal batch; rows are token-major, batch innermost */
  void *q;             /* EPI_QKV: q [M, d]                                    */
  void *kv_a, *kv_b;   /* EPI_QKV: slot(s) [N_tok, B, 2, d]; kv_b may be NULL  */
  int64_t kv_row0;
  int32_t d;
  float *ws;           /* BF16 GEMM split-K workspace (f32, caller-owned device memory,
                          ws_elems floats) or NULL: with a workspace, GEMMs whose tiles
                          fill at most half the SMs split K and reduce the partials in a
                          fixed order (bitwise reproducible)                     */
  int64_t ws_elems;
} stadi_k_epi;

/* out = epilogue(A[M,K] . W[N,K]^T).  BF16 path: K % 64 == 0, N % 64 == 0.
 * Column pairs are accessed as 8-byte vectors: ldo, ldr and gate_bstride must be
 * even (EINVAL otherwise); 16-byte rows take the 16-byte epilogue. */
stadi_status stadi_k_gemm(int32_t dtype, const void *A, const void *W, int32_t M, int32_t N,
                          int32_t K, int32_t epi, const stadi_k_epi *ep, void *stream);

/* As stadi_k_gemm, with the persistent grid capped at max_ctas CTAs (0 = all
 * SMs).  max_ctas < #SMs reproduces the runtime's launch while the occupancy
 * emulator holds SMs (R24): single-CTA tiles on a shrunk grid,
 * and the split-K choice of that grid. */
stadi_status stadi_k_gemm_ex(int32_t dtype, const void *A, const void *W, int32_t M, int32_t N,
                             int32_t K, int32_t epi, const stadi_k_epi *ep, int32_t max_ctas,
                             void *stream);

/* o = softmax(q k^T / sqrt(hd)) v per (batch b, head h).
 * q, o: [Nq * B, H*hd] (row = token*B + b); kv: [Nkv, B, 2, H*hd].
 * BF16 path: hd in {16, 64, 72, 80}. */
stadi_status stadi_k_attention(int32_t dtype, const void *q, const void *kv, void *o, int32_t Nq,
                               int32_t Nkv, int32_t B, int32_t H, int32_t hd, void *stream);

/* y[row] = LayerNorm(x[row]) * (1 + scale[b]) + shift[b], b = row % B (eps 1e-6);
 * x f32 [M, d], y T [M, d]. */
stadi_status stadi_k_ln_modulate(int32_t dtype, const float *x, void *y, int32_t M, int32_t d,
                                 int32_t B, const float *shift, const float *scale,
                                 int32_t bstride, void *stream);

/* 3x3 convolution (pad 1) of the halo-padded input P [h+2, W+2, B, C] (T; row 0 /
 * h+1 are the halo rows, columns 0 / W+1 zero) with Wt [N, Kp] (T, column
 * (ky*3 + kx)*C + c, Kp = 9C rounded up to 64): out[f32] [(oy*Wo + ox)*B + b][N]
 * = conv + bias.  mode 0 stride 1, 1 stride 2, 2 nearest-x2 upsample of P.
 * implicit = 1 (BF16, mode 0, C % 64 == 0): the implicit-GEMM tcgen05 kernel (A
 * tiles TMA-loaded from P); otherwise im2col + GEMM. */
stadi_status stadi_k_conv3x3(int32_t dtype, const void *P, const void *Wt, int32_t h, int32_t W,
                             int32_t B, int32_t C, int32_t N, int32_t mode, int32_t implicit,
                             const float *bias, float *out, void *stream);

/* As stadi_k_conv3x3 with the full EPI_CONV epilogue of the U-Net ResBlock:
 * out[f32] (row stride ep->ldo) = conv + bias + gate[row % B] (time-embedding
 * term, batch stride ep->gate_bstride; NULL = none) + res[row] (f32, row stride
 * ep->ldr; NULL = none); ep->ws / ws_elems: split-K workspace (f32; NULL = allocated
 * per call); other ep fields ignored.  max_ctas as stadi_k_gemm_ex. */
stadi_status stadi_k_conv3x3_ex(int32_t dtype, const void *P, const void *Wt, int32_t h,
                                int32_t W, int32_t B, int32_t C, int32_t N, int32_t mode,
                                int32_t implicit, const stadi_k_epi *ep, int32_t max_ctas,
                                void *stream);

/* Fused CFG + unpatchify + sampler update of an fp32 band x [rows, W, C]
 * (NHWC; Eq. 3, R19 DDPM): eps_raw f32 [tokens * B, ld], token
 * (row/p)*(W/p) + col/p, column ((row%p)*p + col%p)*c_out + ch; with B == 2
 * eps = e0 + guidance (e1 - e0) (R20); x = A x + Bc eps + Cz z, z the element's
 * draw of the R19 generator (key (seed, m), full-image index (row0 + row)*W*C
 * + ...), skipped when Cz == 0. */
stadi_status stadi_k_sampler(float *x, const float *eps_raw, int32_t rows, int32_t W, int32_t C,
                             int32_t p, int32_t c_out, int32_t ld, int32_t B, float guidance,
                             float A, float Bc, float Cz, uint64_t seed, uint32_t m,
                             int32_t row0, void *stream);

/* out[i] = z_m element e0 + i of the R19 generator (Philox4x64-10 key (seed, m),
 * Box-Muller), i < n.  out: f32 device. */
stadi_status stadi_k_ddpm_noise(float *out, int64_t n, uint64_t seed, uint32_t m, int64_t e0,
                                void *stream);

/* GroupNorm(32 groups) of a U-Net band (PAPER.md L80 -- the band's
 * partial sums are the GN exchange payload): x f32 [h, W, B, C] (token-major,
 * batch innermost), B <= 2, C % 32 == 0, C <= 3072.  Step 1 writes the band's
 * partial sums stats f64 [B][32][{sum x, sum x^2}] (caller-owned, device; ws f64
 * [592 * 2 * B * 32] and ticket (32 zero-initialised uint32) are scratch);
 * step 2 normalises with n_total = h * W * C / 32 elements per group (mean =
 * S1 / n, var = max(S2 / n - mean^2, 0)), applies gamma / beta (f32 [C]), SiLU
 * when act != 0, and writes out (T = bf16 or f32 per dtype) either plain [h, W,
 * B, C] (pad == 0) or into the interior of the halo-padded [h+2, W+2, B, C]
 * (pad == 1; the left / right border columns zeroed, halo rows untouched). */
stadi_status stadi_k_groupnorm(int32_t dtype, const float *x, int32_t h, int32_t W, int32_t B,
                               int32_t C, const float *gamma, const float *beta, float eps,
                               int32_t act, int32_t pad, double *stats, double *ws,
                               uint32_t *ticket, void *out, void *stream);

/* Number of kernels launched by this process so far. */
uint64_t stadi_k_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* STADI_KERNELS_H_ */
