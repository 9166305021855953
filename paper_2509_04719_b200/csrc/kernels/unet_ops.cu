// HBM-bound kernels of the patch-parallel U-Net:
// GroupNorm partial statistics of a band (the payload of a GN exchange site,
// PAPER.md L80 "stale activations"), GroupNorm apply (+SiLU) into
// the halo-padded conv-input buffer, im2col of a 3x3 conv (stride 1, stride 2,
// nearest-x2 upsample), channel concat of the skip path and the latent -> padded
// conv_in input.
//
// Activation layout (token-major, batch innermost, as the DiT path):
//   X [h, W, B, C] fp32: element ((y * W + x) * B + b) * C + c
//   P [h + 2, W + 2, B, C] bf16, the conv input with one halo row above / below
//     (filled by the exchange or zero at the image edge) and one zero column
//     left / right: element (((y + 1) * (W + 2) + x + 1) * B + b) * C + c.
#include "../kernels.h"

namespace stadi {

namespace {

constexpr int GN_G = 32;

// ------------------------------------------------------------- GN partials
// out[b][g][0] = sum x, out[b][g][1] = sum x^2 over the band, DETERMINISTIC: one
// block = a chunk of rows; thread t owns float4 channel vector t % nvec of row
// slots t / nvec (all 256 threads busy when nvec < 256), fp32 per thread, reduced
// in smem per (b, channel), then per (b, group) in fp64 into the block's own
// workspace row; the last block to finish (atomic ticket) sums the rows in block
// order and resets the ticket -- the same bits on every run (no fp64 atomics).
__global__ void __launch_bounds__(256) gn_partials_kernel(const float *__restrict__ x, long M,
                                                          int B, int C, int rows_per_block,
                                                          double *__restrict__ ws,
                                                          unsigned *__restrict__ ticket,
                                                          double *__restrict__ out) {
  pdl_wait();
  extern __shared__ float sm[];  // [2 stats][slots][B][C]
  __shared__ bool last;
  const int nvec = C / 4;
  const int slots = nvec >= 256 ? 1 : 256 / nvec;
  const long r0 = (long)blockIdx.x * rows_per_block;
  const long r1 = min(M, r0 + rows_per_block);
  for (int t = threadIdx.x; t < (nvec >= 256 ? nvec : slots * nvec); t += blockDim.x) {
    const int v = t % nvec, slot = t / nvec;
    float4 s1a = make_float4(0.f, 0.f, 0.f, 0.f), s2a = s1a, s1b = s1a, s2b = s1a;
    for (long r = r0 + slot; r < r1; r += slots) {
      const float4 a = reinterpret_cast<const float4 *>(x + r * C)[v];
      if ((r % B) == 0) {
        s1a.x += a.x; s1a.y += a.y; s1a.z += a.z; s1a.w += a.w;
        s2a.x += a.x * a.x; s2a.y += a.y * a.y; s2a.z += a.z * a.z; s2a.w += a.w * a.w;
      } else {
        s1b.x += a.x; s1b.y += a.y; s1b.z += a.z; s1b.w += a.w;
        s2b.x += a.x * a.x; s2b.y += a.y * a.y; s2b.z += a.z * a.z; s2b.w += a.w * a.w;
      }
    }
    float *p1 = sm + ((0 * slots + slot) * B) * C + 4 * v;
    float *p2 = sm + ((1 * slots + slot) * B) * C + 4 * v;
    *reinterpret_cast<float4 *>(p1) = s1a;
    *reinterpret_cast<float4 *>(p2) = s2a;
    if (B > 1) {
      *reinterpret_cast<float4 *>(p1 + C) = s1b;
      *reinterpret_cast<float4 *>(p2 + C) = s2b;
    }
  }
  __syncthreads();
  const int cg = C / GN_G, nst = 2 * B * GN_G;
  for (int jj = threadIdx.x; jj < nst; jj += blockDim.x) {
    const int st = jj / (B * GN_G), b = (jj / GN_G) % B, g = jj % GN_G;
    double acc = 0.0;
    for (int sl = 0; sl < slots; ++sl)
      for (int c = 0; c < cg; ++c) acc += (double)sm[((st * slots + sl) * B + b) * C + g * cg + c];
    ws[(long)blockIdx.x * nst + ((long)b * GN_G + g) * 2 + st] = acc;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int jj = threadIdx.x; jj < nst; jj += blockDim.x) {
    double acc = 0.0;
    for (unsigned k = 0; k < gridDim.x; ++k) acc += __ldcg(ws + (long)k * nst + jj);
    out[jj] = acc;
  }
  if (threadIdx.x == 0) *ticket = 0;  // ready for the next launch (stream-ordered)
}

// ------------------------------------------------------------- GN apply
// y = (x - mean) * rstd * gamma + beta (+ SiLU), mean / var from the sum over the
// G rank segments of the statistics (own fresh + others stale); stats == null:
// plain cast.  pad: write into the halo-padded buffer (interior + zero columns).
template <typename T>
__global__ void __launch_bounds__(256) gn_apply_kernel(
    const float *__restrict__ x, int h, int W, int B, int C, const double *__restrict__ stats,
    int G, double n_total, const float *__restrict__ gamma, const float *__restrict__ beta,
    float eps, int act, int pad, T *__restrict__ out) {
  pdl_wait();
  __shared__ float mu[2 * GN_G], rs[2 * GN_G];
  if (stats) {
    for (int j = threadIdx.x; j < B * GN_G; j += blockDim.x) {
      double s1 = 0, s2 = 0;
      for (int q = 0; q < G; ++q) {
        s1 += stats[((long)q * B * GN_G + j) * 2 + 0];
        s2 += stats[((long)q * B * GN_G + j) * 2 + 1];
      }
      const double m = s1 / n_total;
      const double var = fmax(s2 / n_total - m * m, 0.0);  // R17 clamp
      mu[j] = (float)m;
      rs[j] = (float)(1.0 / sqrt(var + (double)eps));
    }
  }
  __syncthreads();
  const int nvec = C / 4, cg = C / GN_G;
  const long total = (long)h * W * B * nvec;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int v = (int)(i % nvec);
    const long row = i / nvec;  // (y * W + x) * B + b
    const int b = (int)(row % B);
    float4 a = reinterpret_cast<const float4 *>(x + row * C)[v];
    float e[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = 4 * v + k;
      float y = e[k];
      if (stats) {
        const int j = b * GN_G + c / cg;
        y = (y - mu[j]) * rs[j] * gamma[c] + beta[c];
      }
      if (act) y = silu(y);
      e[k] = y;
    }
    long orow = row;
    if (pad) {
      const long pix = row / B;
      const int yy = (int)(pix / W), xx = (int)(pix % W);
      orow = (((long)(yy + 1) * (W + 2) + xx + 1) * B + b);
    }
    T *o = out + orow * C + 4 * v;
    if constexpr (sizeof(T) == 2) {  // one 8-byte store of 4 bf16
      __nv_bfloat162 lo = __floats2bfloat162_rn(e[0], e[1]), hi = __floats2bfloat162_rn(e[2], e[3]);
      *reinterpret_cast<uint2 *>(o) =
          make_uint2(*reinterpret_cast<uint32_t *>(&lo), *reinterpret_cast<uint32_t *>(&hi));
    } else {
      *reinterpret_cast<float4 *>(o) = make_float4(e[0], e[1], e[2], e[3]);
    }
    if (pad) {  // zero the left / right border columns of this row
      const long pix = row / B;
      const int yy = (int)(pix / W), xx = (int)(pix % W);
      if (xx == 0 || xx == W - 1) {
        const long brow = (((long)(yy + 1) * (W + 2) + (xx == 0 ? 0 : W + 1)) * B + b);
        T *z = out + brow * C + 4 * v;
        z[0] = z[1] = z[2] = z[3] = from_f<T>(0.f);
      }
    }
  }
}

// latent band x [h, W, Cl] fp32 -> padded conv_in input [h+2, W+2, B, Cl] (B copies)
template <typename T>
__global__ void latent_pad_kernel(const float *__restrict__ x, int h, int W, int Cl, int B,
                                  T *__restrict__ out) {
  pdl_wait();
  const long total = (long)(h + 2) * (W + 2) * B * Cl;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int c = (int)(i % Cl);
    const long pix = i / Cl / B;
    const int yy = (int)(pix / (W + 2)), xx = (int)(pix % (W + 2));
    if (yy == 0 || yy == h + 1) continue;  // halo rows belong to the exchange
    float v = 0.f;
    if (xx >= 1 && xx <= W) v = x[((long)(yy - 1) * W + (xx - 1)) * Cl + c];
    out[i] = from_f<T>(v);
  }
}

// ------------------------------------------------------------- im2col
// A[((oy * Wo + ox) * B + b)][(ky * 3 + kx) * C + c] from the padded input
// (mode 0: stride 1; 1: stride 2; 2: nearest-x2 upsample of the input).
// Columns >= 9C up to Kp are zero.  V = elements per thread (8 if C % 8 == 0).
template <typename T, int V>
__global__ void __launch_bounds__(256) im2col_kernel(const T *__restrict__ P, int hin, int Win,
                                                     int B, int C, int mode, int ho, int wo,
                                                     int Kp, T *__restrict__ A) {
  pdl_wait();
  const int kv = Kp / V;  // vectors per A row
  const long total = (long)ho * wo * B * kv;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int k0 = (int)(i % kv) * V;
    const long row = i / kv;
    const int b = (int)(row % B);
    const long pix = row / B;
    const int oy = (int)(pix / wo), ox = (int)(pix % wo);
    T *dst = A + row * Kp + k0;
    const int tap = k0 / C, c = k0 % C;
    bool zero = tap >= 9;
    long src = 0;
    if (!zero) {
      const int ky = tap / 3, kx = tap % 3;
      int py, px;
      if (mode == 0) {
        py = oy + ky;
        px = ox + kx;
      } else if (mode == 1) {
        py = 2 * oy + ky;
        px = 2 * ox + kx;
      } else {
        const int Y = oy + ky, X = ox + kx;  // hi-res padded coordinates
        if (X == 0 || X == 2 * Win + 1) {
          zero = true;
          py = px = 0;
        } else {
          py = Y == 0 ? 0 : (Y == 2 * hin + 1 ? hin + 1 : 1 + (Y - 1) / 2);
          px = 1 + (X - 1) / 2;
        }
      }
      src = (((long)py * (Win + 2) + px) * B + b) * C + c;
    }
    if constexpr (V == 8) {
      uint4 v = make_uint4(0, 0, 0, 0);
      if (!zero) v = *reinterpret_cast<const uint4 *>(P + src);
      *reinterpret_cast<uint4 *>(dst) = v;
    } else {
      dst[0] = zero ? from_f<T>(0.f) : P[src];
    }
  }
}

// ------------------------------------------------------------- halo rows
// The two halo rows of the padded conv input P [h+2, W+2, B, C]: row 0 = `above`
// (W * B * C elements, or zeros at the image's top edge when null), row h+1 =
// `below` (or zeros), and the four corner cells zero.  One launch replaces two
// copies and four memsets per conv.  16-byte vectors (C * esz % 16 == 0) when aligned.
template <typename T>
__global__ void __launch_bounds__(256) halo_fill_kernel(T *__restrict__ P, int h, int W, int B,
                                                        int C, const T *__restrict__ above,
                                                        const T *__restrict__ below) {
  pdl_wait();
  const long rowe = (long)(W + 2) * B * C;        // elements of one padded row
  const long inner = (long)W * B * C;             // interior elements of a row
  const long cell = (long)B * C;
  constexpr int V = 16 / sizeof(T);
  const bool vec = (cell % V) == 0;
  const long n = vec ? 2 * rowe / V : 2 * rowe;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    const long e = vec ? i * V : i;               // element offset within the two rows
    const int r = (int)(e / rowe);                 // 0: top halo, 1: bottom halo
    const long off = e % rowe;                     // within the padded row
    const long x = off - cell;                     // within the interior
    const T *src = r ? below : above;
    T *dst = P + (r ? (long)(h + 1) * rowe : 0) + off;
    const bool interior = x >= 0 && x < inner;
    if (vec) {
      uint4 v = make_uint4(0, 0, 0, 0);
      if (interior && src) v = *reinterpret_cast<const uint4 *>(src + x);
      *reinterpret_cast<uint4 *>(dst) = v;
    } else {
      *dst = (interior && src) ? src[x] : from_f<T>(0.f);
    }
  }
}

// ------------------------------------------------------------- concat
__global__ void concat_kernel(const float *__restrict__ a, int Ca, const float *__restrict__ b,
                              int Cb, long M, float *__restrict__ out) {
  pdl_wait();
  const int C = Ca + Cb;
  const long total = M * (C / 4);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int v = (int)(i % (C / 4));
    const long r = i / (C / 4);
    const int c = 4 * v;
    float4 x = c < Ca ? reinterpret_cast<const float4 *>(a + r * Ca)[v]
                      : reinterpret_cast<const float4 *>(b + r * Cb)[(c - Ca) / 4];
    reinterpret_cast<float4 *>(out + r * C)[v] = x;
  }
}

inline unsigned grid_for(long work, int per_block = 256) {
  long g = (work + per_block - 1) / per_block;
  return (unsigned)std::min<long>(std::max<long>(g, 1), 148L * 16);
}

}  // namespace

cudaError_t gn_partials(const float *x, long M, int B, int C, double *out, double *ws,
                        unsigned *ticket, cudaStream_t s) {
  if (C % (4 * GN_G) && C % 4) return cudaErrorInvalidValue;
  if (B > 2 || C % 4 || C % GN_G || !ws || !ticket) return cudaErrorInvalidValue;
  if (M == 0) return cudaMemsetAsync(out, 0, (size_t)B * GN_G * 2 * sizeof(double), s);
  const int blocks = (int)std::min<long>(GN_PARTIAL_BLOCKS, M);
  int rpb = (int)((M + blocks - 1) / blocks);
  const int nb = (int)((M + rpb - 1) / rpb);
  const int nvec = C / 4, slots = nvec >= 256 ? 1 : 256 / nvec;
  const size_t smem = (size_t)2 * slots * B * C * sizeof(float);
  const cudaError_t el = launch_pdl(gn_partials_kernel, dim3(nb), dim3(256), smem, s, x, M, B, C,
                                    rpb, ws, ticket, out);
  ++g_launches;
  return el;
}

template <typename T>
cudaError_t gn_apply(const float *x, int h, int W, int B, int C, const double *stats, int G,
                     double n_total, const float *gamma, const float *beta, float eps, int act,
                     int pad, T *out, cudaStream_t s) {
  if (C % 4 || (stats && C % GN_G) || B > 2) return cudaErrorInvalidValue;
  const long work = (long)h * W * B * (C / 4);
  if (work == 0) return cudaSuccess;
  const cudaError_t el = launch_pdl(gn_apply_kernel<T>, dim3(grid_for(work)), dim3(256), 0, s, x,
                                    h, W, B, C, stats, G, n_total, gamma, beta, eps, act, pad, out);
  ++g_launches;
  return el;
}
template cudaError_t gn_apply<bf16>(const float *, int, int, int, int, const double *, int,
                                    double, const float *, const float *, float, int, int, bf16 *,
                                    cudaStream_t);
template cudaError_t gn_apply<float>(const float *, int, int, int, int, const double *, int,
                                     double, const float *, const float *, float, int, int,
                                     float *, cudaStream_t);

template <typename T>
cudaError_t halo_fill(T *P, int h, int W, int B, int C, const T *above, const T *below,
                      cudaStream_t s) {
  const long rowe = (long)(W + 2) * B * C;
  const long work = 2 * rowe / (((long)B * C) % (16 / sizeof(T)) == 0 ? 16 / sizeof(T) : 1);
  const cudaError_t el = launch_pdl(halo_fill_kernel<T>, dim3(grid_for(work)), dim3(256), 0, s, P,
                                    h, W, B, C, above, below);
  ++g_launches;
  return el;
}
template cudaError_t halo_fill<bf16>(bf16 *, int, int, int, int, const bf16 *, const bf16 *,
                                     cudaStream_t);
template cudaError_t halo_fill<float>(float *, int, int, int, int, const float *, const float *,
                                      cudaStream_t);

template <typename T>
cudaError_t latent_pad(const float *x, int h, int W, int Cl, int B, T *out, cudaStream_t s) {
  const long work = (long)(h + 2) * (W + 2) * B * Cl;
  const cudaError_t el = launch_pdl(latent_pad_kernel<T>, dim3(grid_for(work)), dim3(256), 0, s, x,
                                    h, W, Cl, B, out);
  ++g_launches;
  return el;
}
template cudaError_t latent_pad<bf16>(const float *, int, int, int, int, bf16 *, cudaStream_t);
template cudaError_t latent_pad<float>(const float *, int, int, int, int, float *, cudaStream_t);

template <typename T>
cudaError_t im2col(const T *P, int hin, int Win, int B, int C, int mode, int Kp, T *A,
                   cudaStream_t s) {
  const int ho = mode == 1 ? hin / 2 : (mode == 2 ? 2 * hin : hin);
  const int wo = mode == 1 ? Win / 2 : (mode == 2 ? 2 * Win : Win);
  if (Kp < 9 * C) return cudaErrorInvalidValue;
  if (C % 8 == 0 && Kp % 8 == 0 && sizeof(T) == 2) {
    const long work = (long)ho * wo * B * (Kp / 8);
    const cudaError_t el = launch_pdl(im2col_kernel<T, 8>, dim3(grid_for(work)), dim3(256), 0, s,
                                      P, hin, Win, B, C, mode, ho, wo, Kp, A);
    if (el != cudaSuccess) return el;
  } else {
    const long work = (long)ho * wo * B * Kp;
    const cudaError_t el = launch_pdl(im2col_kernel<T, 1>, dim3(grid_for(work)), dim3(256), 0, s,
                                      P, hin, Win, B, C, mode, ho, wo, Kp, A);
    if (el != cudaSuccess) return el;
  }
  ++g_launches;
  return cudaGetLastError();
}
template cudaError_t im2col<bf16>(const bf16 *, int, int, int, int, int, int, bf16 *,
                                  cudaStream_t);
template cudaError_t im2col<float>(const float *, int, int, int, int, int, int, float *,
                                   cudaStream_t);

cudaError_t concat_channels(const float *a, int Ca, const float *b, int Cb, long M, float *out,
                            cudaStream_t s) {
  if (Ca % 4 || Cb % 4) return cudaErrorInvalidValue;
  const long work = M * ((Ca + Cb) / 4);
  if (work == 0) return cudaSuccess;
  const cudaError_t el = launch_pdl(concat_kernel, dim3(grid_for(work)), dim3(256), 0, s, a, Ca, b,
                                    Cb, M, out);
  ++g_launches;
  return el;
}

}  // namespace stadi
