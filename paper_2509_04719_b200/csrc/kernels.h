// Host launch functions of the libstadi kernels (all stream-ordered).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "device.cuh"

namespace stadi {

// Global launch counter (kernels launched by this process).
extern unsigned long long g_launches;

// ---- GEMM  out = epilogue(A[M,K] . W[N,K]^T) ------------------------------
// SIMT fp32-accumulate GEMM (the fp32 debug build, and tiny conditioning GEMMs).
template <typename T>
cudaError_t simt_gemm(const T *A, const T *W, int M, int N, int K, int epi, const EpiParams &ep,
                      cudaStream_t s);
// tcgen05 + TMA bf16 GEMM (persistent, warp-specialised).  Requires K % 64 == 0,
// N % 64 == 0.  max_ctas bounds the grid (SMs not pinned by the emulator).
cudaError_t tc_gemm_bf16(const bf16 *A, const bf16 *W, int M, int N, int K, int epi,
                         const EpiParams &ep, int max_ctas, cudaStream_t s);
// Implicit-GEMM 3x3 conv from the halo-padded input P [h+2, W+2, B, C]: mode 0 stride
// 1, mode 1 stride 2 (h, W even); C % 64 == 0, (output width)*B a divisor or multiple of
// 128 (tc_conv_implicit_ok); epi EPI_CONV or EPI_F32.
bool tc_conv_implicit_ok(int h, int W, int B, int C, int N, int mode);
cudaError_t tc_conv3x3_bf16(const bf16 *P, const bf16 *Wt, int h, int W, int B, int C, int N,
                            int epi, const EpiParams &ep, int max_ctas, cudaStream_t s,
                            int mode = 0);
// Nearest-x2 upsample of the halo-padded P [h+2, W+2, B, C] into the halo-padded
// U [2h+2, 2W+2, B, C]: U row Y <- P row 0 (Y = 0), h+1 (Y = 2h+1), else 1 + (Y-1)/2;
// U column X <- P column 1 + (X-1)/2, zero for X = 0 / 2W+1 (the upsample conv's input,
// so the conv runs as an implicit stride-1 conv instead of over a 9x im2col buffer).
template <typename T>
cudaError_t upsample_pad(const T *P, int h, int W, int B, int C, T *U, cudaStream_t s);

// ---- attention  o = softmax(q k^T / sqrt(hd)) v  per (batch b, head h) ------
// q, o: [Nq * B, H*hd] (row = token*B + b);  kv: [Nkv, B, 2, H*hd] (K then V).
template <typename T>
cudaError_t simt_attention(const T *q, const T *kv, T *o, int Nq, int Nkv, int B, int H, int hd,
                           cudaStream_t s);
cudaError_t tc_attention_bf16(const bf16 *q, const bf16 *kv, bf16 *o, int Nq, int Nkv, int B,
                              int H, int hd, cudaStream_t s);
bool tc_attention_supported(int hd);

// ---- elementwise / normalisation -------------------------------------------
// y[row] = LN(x[row]) * (1 + scale[b]) + shift[b]   (b = row % B); do_norm = 0: y = x
// eps: 1e-6 (DiT, no affine) or 1e-5 (U-Net LayerNorm with affine: scale = w - 1,
// shift = b, mod_bstride = 0).
template <typename T>
cudaError_t ln_modulate(const float *x, T *y, int M, int d, int B, const float *shift,
                        const float *scale, int mod_bstride, int do_norm, cudaStream_t s,
                        float eps = 1e-6f);
// Patchify a latent band + Linear(p*p*C -> d) + bias + positional embedding,
// written for every batch row: x_res[(i*B+b), :].
cudaError_t patch_embed(const float *x_band, int rows, int W, int C, int p, const float *w,
                        const float *b, const float *pos_rows, int d, int B, float *x_res,
                        cudaStream_t s);
// CFG combine + unpatchify + sampler update of the band:
//   x = A x + Bc eps (+ Cz z_m when Cz != 0: R19 DDPM, z_m drawn in-kernel by
//   Philox4x64-10 with key (seed, m) at the element's full-image index, the
//   band starting at latent row row0).  eps_raw row stride = ld (>= p*p*c_out).
//   The key is *seed_dev when seed_dev != NULL (read at run time, so a captured
//   CUDA graph serves every request), else `seed`.  hist != NULL (R34 multistep
//   DPM-Solver-2): eps -> c1 eps + c2 hist (hist = the band's previous combined eps;
//   c2 == 0: first step), and hist <- eps.
cudaError_t sampler_update(float *x_band, const float *eps_raw, int rows, int W, int C, int p,
                           int c_out, int ld, int B, float guidance, float A, float Bc,
                           float Cz, uint64_t seed, const uint64_t *seed_dev, uint32_t m, int row0,
                           cudaStream_t s, float *hist = nullptr, float c1 = 1.f, float c2 = 0.f);
// z_m elements [e0, e0 + n) of the R19 generator (parity tests).
cudaError_t philox_normal_fill(float *out, long n, uint64_t seed, uint32_t m, long e0,
                               cudaStream_t s);
// Conditioning helpers
cudaError_t silu_inplace(float *x, long n, cudaStream_t s);
template <typename T>
cudaError_t class_cond(const float *temb, const float *table, const int *labels, int n_t, int B,
                       int d, T *out, cudaStream_t s);
template <typename T>
cudaError_t silu_cast(const float *x, T *y, long n, cudaStream_t s);
template <typename T>
cudaError_t cast_f32(const float *x, T *y, long n, cudaStream_t s);
cudaError_t pixart_mods(const float *t0, const float *temb, const float *sst_all,
                        const float *final_sst, int n_t, int B, int depth, int d, float *mod,
                        float *fmod, cudaStream_t s);

// ---- U-Net band kernels (unet_ops.cu): X = [h, W, B, C] fp32 token-major,
// P = [h+2, W+2, B, C] halo-padded conv input (see unet_ops.cu) --------------
// GroupNorm partial sums of the band: out[b][g][{S1, S2}] (fp64), reduced across
// blocks in a fixed order (bitwise reproducible): ws = GN_PARTIAL_BLOCKS * 2 * B * 32
// doubles of workspace, ticket = 32 zero-initialised unsigned (reset by the kernel);
// one (ws, ticket) pair per stream.
// out2 / out3 (optional): further copies of out (the exchange slots).  C <= 3072.
constexpr int GN_PARTIAL_BLOCKS = 592;
cudaError_t gn_partials(const float *x, long M, int B, int C, double *out, double *ws,
                        unsigned *ticket, cudaStream_t s, double *out2 = nullptr,
                        double *out3 = nullptr);
// Halo rows of the padded conv input P [h+2, W+2, B, C]: row 0 <- above, row h+1
// <- below (W*B*C elements each; NULL = zeros at the image edge), corners zero.
template <typename T>
cudaError_t halo_fill(T *P, int h, int W, int B, int C, const T *above, const T *below,
                      cudaStream_t s);
// GroupNorm with the statistics summed over G rank segments [G][B][32][2]
// (stats == null: plain cast), optional SiLU, pad = write into P's interior.
template <typename T>
cudaError_t gn_apply(const float *x, int h, int W, int B, int C, const double *stats, int G,
                     double n_total, const float *gamma, const float *beta, float eps, int act,
                     int pad, T *out, cudaStream_t s, int zero_halo = 0);
// latent band [h, W, Cl] -> P (B copies; halo rows untouched unless zero_halo)
// zero_halo (pad only): bit 0 zeroes halo row 0, bit 1 row h + 1 (image-edge rows of a
// band, so the conv of a band without neighbours needs no halo_fill)
template <typename T>
cudaError_t latent_pad(const float *x, int h, int W, int Cl, int B, T *out, cudaStream_t s,
                       int zero_halo = 0);
// 3x3 conv im2col from P: mode 0 stride 1, 1 stride 2, 2 nearest-x2 upsample.
// A [(oy*Wo + ox)*B + b][Kp], column (ky*3 + kx)*C + c, zero beyond 9C.
template <typename T>
cudaError_t im2col(const T *P, int hin, int Win, int B, int C, int mode, int Kp, T *A,
                   cudaStream_t s);
cudaError_t concat_channels(const float *a, int Ca, const float *b, int Cb, long M, float *out,
                            cudaStream_t s);

// ---- occupancy emulator ---------------------------------
cudaError_t emulator_launch(int n_ctas, volatile int *stop_flag, cudaStream_t s);
// Force-load every tcgen05 GEMM / attention kernel instance (lazy loading must
// not happen while the occupancy emulator's kernel is resident: deadlock).
cudaError_t tc_gemm_preload();
cudaError_t tc_attention_preload();
// SMs the emulator takes for pct% occupancy: ceil(pct * SMs / 100) rounded up to
// whole TPCs (even).
int emulator_ctas(int pct, int num_sms);

}  // namespace stadi
