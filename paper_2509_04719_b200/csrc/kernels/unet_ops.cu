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
// out[b][g][0] = sum x, out[b][g][1] = sum x^2 over the band, DETERMINISTIC (the
// same bits on every run: fixed per-thread row sets, fixed-order reductions, no
// floating-point atomics).  One block = a chunk of rpb consecutive rows (rpb even,
// so a row's batch index is its parity when B = 2), <= GNP_MAXB blocks:
//   thread t owns NV float4 channel vectors v = t % nvec (+ 256 k) of the rows
//   r0 + slot + i slots (slot = t / nvec; one slot when nvec >= 256), loads UNR
//   rows at a time (independent loads in flight: the band is latency-, not
//   bandwidth-bound otherwise) and accumulates fp32 sums per (batch, channel);
//   the block folds the slots, then two threads per (statistic, batch, group)
//   output sum half the group's channels each in fp64 (one shuffle) into the
//   block's workspace row.
// Cross-block, two fixed-order levels: the last block of each set of GNP_SET
// blocks (set ticket) sums the set's rows into a set row, the last set to finish
// (global ticket) sums the set rows and writes out and, optionally, out2 / out3
// (the exchange slots, saving two copies); tickets reset for the next launch.
// ticket: 1 + GNP_MAXB / GNP_SET zero-initialised unsigned.
constexpr int GNP_THREADS = 256;
constexpr int GNP_MAXB = 296;  // blocks per launch (2 per SM)
constexpr int GNP_SET = 16;    // blocks per first-level reduction set
constexpr int GNP_SETROW0 = 320;  // workspace row of set 0 (after the block rows)

// two threads per output: sum rows [k0, k1) of ws (row stride nst) for output o,
// this thread taking every other row (hf) -- fixed order, one load wave
template <int MAXR>
__device__ __forceinline__ double gnp_sum_rows(const double *ws, int nst, int o, int hf, int k0,
                                               int k1) {
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < MAXR; ++i) {
    const int k = k0 + 2 * i + hf;
    if (k < k1) acc += __ldcg(ws + (long)k * nst + o);
  }
  return acc + __shfl_xor_sync(0xffffffffu, acc, 1);
}

template <int NV>
__global__ void __launch_bounds__(GNP_THREADS) gn_partials_kernel(
    const float *__restrict__ x, int M, int B, int C, int rpb, double *__restrict__ ws,
    unsigned *__restrict__ ticket, double *__restrict__ out, double *__restrict__ out2,
    double *__restrict__ out3) {
  constexpr int UNR = NV == 1 ? 8 : 4;
  extern __shared__ float sm[];  // [2 stats][slots][B][C]
  __shared__ bool last;
  pdl_wait();
  const int nvec = C / 4;
  const int slots = nvec >= GNP_THREADS ? 1 : GNP_THREADS / nvec;
  const int r0 = blockIdx.x * rpb, r1 = min(M, r0 + rpb);
  const int t = threadIdx.x;
  if (t < slots * nvec || nvec >= GNP_THREADS) {
    const int slot = nvec >= GNP_THREADS ? 0 : t / nvec;
    const int v0 = nvec >= GNP_THREADS ? t : t % nvec;
    float4 s1[2][NV], s2[2][NV];
#pragma unroll
    for (int bb = 0; bb < 2; ++bb)
#pragma unroll
      for (int k = 0; k < NV; ++k) s1[bb][k] = s2[bb][k] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int rb = r0 + slot; rb < r1; rb += UNR * slots) {
      float4 a[UNR][NV];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int r = rb + u * slots;
        const float4 *row = reinterpret_cast<const float4 *>(x + (long)r * C);
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int v = v0 + k * GNP_THREADS;
          a[u][k] = (r < r1 && v < nvec) ? row[v] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const bool odd = B == 2 && ((rb + u * slots) & 1);
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          auto add = [&](float4 &p, float4 &q) {
            const float4 e = a[u][k];
            p.x += e.x; p.y += e.y; p.z += e.z; p.w += e.w;
            q.x += e.x * e.x; q.y += e.y * e.y; q.z += e.z * e.z; q.w += e.w * e.w;
          };
          if (odd) add(s1[1][k], s2[1][k]);
          else add(s1[0][k], s2[0][k]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int v = v0 + k * GNP_THREADS;
      if (v >= nvec) break;
#pragma unroll
      for (int bb = 0; bb < 2; ++bb) {
        if (bb >= B) break;
        *reinterpret_cast<float4 *>(sm + ((0 * slots + slot) * B + bb) * C + 4 * v) = s1[bb][k];
        *reinterpret_cast<float4 *>(sm + ((1 * slots + slot) * B + bb) * C + 4 * v) = s2[bb][k];
      }
    }
  }
  __syncthreads();
  // slots -> slot 0 per (statistic, batch, channel), fixed order
  if (slots > 1) {
    for (int e = t; e < 2 * B * C; e += GNP_THREADS) {
      const int st = e / (B * C), rem = e % (B * C);
      float acc = sm[(st * slots) * B * C + rem];
      for (int sl = 1; sl < slots; ++sl) acc += sm[(st * slots + sl) * B * C + rem];
      sm[(st * slots) * B * C + rem] = acc;
    }
    __syncthreads();
  }
  // per (statistic, batch, group): two threads per output, each half the group's
  // channels in fp64, combined by one shuffle
  const int cg = C / GN_G, nst = 2 * B * GN_G, half = (cg + 1) / 2;
  const int o = t >> 1, hf = t & 1;  // o = (b * 32 + g) * 2 + st
  if (o < nst) {
    const int st = o & 1, g = (o >> 1) % GN_G, bb = (o >> 1) / GN_G;
    const float *src = sm + (st * slots * B + bb) * C + g * cg;
    double acc = 0.0;
    for (int c = hf * half; c < min(cg, (hf + 1) * half); ++c) acc += (double)src[c];
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (hf == 0) ws[(long)blockIdx.x * nst + o] = acc;
  }
  // level 1: the last block of this set sums the set's block rows
  const int set = blockIdx.x / GNP_SET, nsets = (gridDim.x + GNP_SET - 1) / GNP_SET;
  const int k0 = set * GNP_SET, k1 = min((int)gridDim.x, k0 + GNP_SET);
  __threadfence();
  __syncthreads();
  if (t == 0) last = atomicAdd(&ticket[1 + set], 1u) == (unsigned)(k1 - k0 - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (o < nst) {
    const double acc = gnp_sum_rows<GNP_SET / 2>(ws, nst, o, hf, k0, k1);
    if (hf == 0) ws[(long)(GNP_SETROW0 + set) * nst + o] = acc;
  }
  __threadfence();
  __syncthreads();
  if (t == 0) {
    ticket[1 + set] = 0;
    last = atomicAdd(&ticket[0], 1u) == (unsigned)(nsets - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // level 2: the last set sums the set rows
  if (o < nst) {
    const double acc = gnp_sum_rows<(GNP_MAXB / GNP_SET + 2) / 2>(ws, nst, o, hf, GNP_SETROW0,
                                                                GNP_SETROW0 + nsets);
    if (hf == 0) {
      out[o] = acc;
      if (out2) out2[o] = acc;
      if (out3) out3[o] = acc;
    }
  }
  if (t == 0) ticket[0] = 0;  // ready for the next launch (stream-ordered)
}

// ------------------------------------------------------------- GN apply
// y = (x - mean) * (rstd * gamma) + beta (+ SiLU), mean / var from the sum over the
// G rank segments of the statistics (own fresh + others stale); stats == null:
// plain cast.  pad: write into the halo-padded buffer (interior + zero columns).
// One block = a chunk of rpb rows (pixel, batch); its (row, float4) elements are
// walked flat, GNA_UNR per thread in flight, 32-bit indexing; the per-(batch,
// channel) mean and scale live in shared memory (dynamic: (2 B + 1) C floats).
constexpr int GNA_THREADS = 256;
constexpr int GNA_UNR = 4;
// SiLU of the GN output: bf16 output -> x (1 + tanh(x / 2)) / 2 with the single-MUFU
// tanh.approx (rel. error ~2^-11, 4x below the bf16 rounding of the result); fp32 (the
// <= 1e-4 debug build) -> the accurate x / (1 + e^-x)
template <typename T>
__device__ __forceinline__ float silu_out(float x) {
  if constexpr (sizeof(T) == 2) {
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
    return 0.5f * x * (1.f + t);
  } else {
    return silu(x);
  }
}
template <typename T>
__global__ void __launch_bounds__(GNA_THREADS) gn_apply_kernel(
    const float *__restrict__ x, int h, int W, int B, int C, int rpb,
    const double *__restrict__ stats, int G, double n_total, const float *__restrict__ gamma,
    const float *__restrict__ beta, float eps, int act, int pad, T *__restrict__ out,
    int zero_halo) {
  extern __shared__ float gsm[];  // mu [B][C], sc [B][C], beta [C]
  __shared__ float mu_g[2 * GN_G], rs_g[2 * GN_G];
  float *mu_c = gsm, *sc_c = gsm + B * C, *be_c = gsm + 2 * B * C;
  pdl_wait();
  const int cg = C / GN_G;
  if (stats) {
    for (int j = threadIdx.x; j < B * GN_G; j += blockDim.x) {
      double s1 = 0, s2 = 0;
      for (int q = 0; q < G; ++q) {
        s1 += stats[((long)q * B * GN_G + j) * 2 + 0];
        s2 += stats[((long)q * B * GN_G + j) * 2 + 1];
      }
      const double m = s1 / n_total;
      const double var = fmax(s2 / n_total - m * m, 0.0);  // R17 clamp
      mu_g[j] = (float)m;
      rs_g[j] = (float)(1.0 / sqrt(var + (double)eps));
    }
    __syncthreads();
    for (int j = threadIdx.x; j < B * C; j += blockDim.x) {
      const int bb = j / C, c = j % C, gj = bb * GN_G + c / cg;
      mu_c[j] = mu_g[gj];
      sc_c[j] = rs_g[gj] * gamma[c];
    }
    for (int c = threadIdx.x; c < C; c += blockDim.x) be_c[c] = beta[c];
    __syncthreads();
  }
  const int nvec = C / 4, M = h * W * B;
  const int r0 = blockIdx.x * rpb, r1 = min(M, r0 + rpb);
  // thread -> fixed float4 channel vector(s) v0 (+ 256 k), rows r0 + slot + i slots:
  // no per-element index division; GNA_UNR rows of loads in flight
  const int t = threadIdx.x;
  const int slots = nvec >= GNA_THREADS ? 1 : GNA_THREADS / nvec;
  const bool busy = nvec >= GNA_THREADS || t < slots * nvec;
  const int slot = nvec >= GNA_THREADS ? 0 : t / nvec;
  const int v0 = nvec >= GNA_THREADS ? t : t % nvec;
  for (int v = v0; busy && v < nvec; v += GNA_THREADS) {
    for (int rb = r0 + slot; rb < r1; rb += GNA_UNR * slots) {
      float4 a[GNA_UNR];
#pragma unroll
      for (int u = 0; u < GNA_UNR; ++u) {
        const int row = rb + u * slots;
        a[u] = row < r1 ? reinterpret_cast<const float4 *>(x + (long)row * C)[v]
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < GNA_UNR; ++u) {
        const int row = rb + u * slots;
        if (row >= r1) break;
        const int bb = B == 2 ? (row & 1) : 0;
        float y[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
        if (stats) {
          const float4 m = *reinterpret_cast<const float4 *>(mu_c + bb * C + 4 * v);
          const float4 sc = *reinterpret_cast<const float4 *>(sc_c + bb * C + 4 * v);
          const float4 be = *reinterpret_cast<const float4 *>(be_c + 4 * v);
          y[0] = (y[0] - m.x) * sc.x + be.x;
          y[1] = (y[1] - m.y) * sc.y + be.y;
          y[2] = (y[2] - m.z) * sc.z + be.z;
          y[3] = (y[3] - m.w) * sc.w + be.w;
        }
        if (act) {
#pragma unroll
          for (int k = 0; k < 4; ++k) y[k] = silu_out<T>(y[k]);
        }
        long orow = row;
        if (pad) {
          const int pix = B == 2 ? (row >> 1) : row, yy = pix / W, xx = pix - yy * W;
          orow = ((long)(yy + 1) * (W + 2) + xx + 1) * B + bb;
        }
        T *o = out + orow * C + 4 * v;
        if constexpr (sizeof(T) == 2) {  // one 8-byte store of 4 bf16
          __nv_bfloat162 lo = __floats2bfloat162_rn(y[0], y[1]),
                         hi = __floats2bfloat162_rn(y[2], y[3]);
          *reinterpret_cast<uint2 *>(o) =
              make_uint2(*reinterpret_cast<uint32_t *>(&lo), *reinterpret_cast<uint32_t *>(&hi));
        } else {
          *reinterpret_cast<float4 *>(o) = make_float4(y[0], y[1], y[2], y[3]);
        }
      }
    }
  }
  if (pad && zero_halo) {  // image-edge halo rows (bit 0: row 0, bit 1: row h + 1), corners too
    const int rowv = (W + 2) * B * nvec;
    for (int e = blockIdx.x * GNA_THREADS + threadIdx.x; e < 2 * rowv;
         e += gridDim.x * GNA_THREADS) {
      const int r = e / rowv;
      if (!((zero_halo >> r) & 1)) continue;
      T *z = out + ((long)(r ? h + 1 : 0) * (W + 2) * B) * C + 4 * (long)(e % rowv);
      z[0] = z[1] = z[2] = z[3] = from_f<T>(0.f);
    }
  }
  if (pad) {  // zero the left / right border cells of the chunk's image rows
    const int p0 = r0 / B, p1 = (r1 - 1) / B;  // pixel range (inclusive)
    const int y0 = p0 / W, ny = p1 / W - y0 + 1;
    const int nz = ny * 2 * B * nvec;
    for (int e = threadIdx.x; e < nz; e += GNA_THREADS) {
      const int cand = e / (B * nvec), rem = e % (B * nvec);
      const int yy = y0 + cand / 2, side = cand & 1;
      const int p = yy * W + (side ? W - 1 : 0);
      if (p < p0 || p > p1) continue;
      const int bb = rem / nvec, v = rem % nvec;
      T *z = out + (((long)(yy + 1) * (W + 2) + (side ? W + 1 : 0)) * B + bb) * C + 4 * v;
      z[0] = z[1] = z[2] = z[3] = from_f<T>(0.f);
    }
  }
}

// latent band x [h, W, Cl] fp32 -> padded conv_in input [h+2, W+2, B, Cl] (B copies)
template <typename T>
__global__ void latent_pad_kernel(const float *__restrict__ x, int h, int W, int Cl, int B,
                                  T *__restrict__ out, int zero_halo) {
  pdl_wait();
  const long total = (long)(h + 2) * (W + 2) * B * Cl;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int c = (int)(i % Cl);
    const long pix = i / Cl / B;
    const int yy = (int)(pix / (W + 2)), xx = (int)(pix % (W + 2));
    // halo rows belong to the exchange, except image-edge rows (zero_halo bit 0 / 1)
    if ((yy == 0 && !(zero_halo & 1)) || (yy == h + 1 && !(zero_halo & 2))) continue;
    float v = 0.f;
    if (yy == 0 || yy == h + 1) {
      out[i] = from_f<T>(0.f);
      continue;
    }
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

// ------------------------------------------------------------- nearest-x2 upsample
// U [2h+2, 2W+2, B, C] from P [h+2, W+2, B, C] (see kernels.h), 16-byte vectors
template <typename T>
__global__ void __launch_bounds__(256) upsample_pad_kernel(const T *__restrict__ P, int h, int W,
                                                           int B, int C, T *__restrict__ U) {
  pdl_wait();
  constexpr int V = 16 / sizeof(T);
  const int cv = C / V;                                   // vectors per (pixel, batch)
  const int Wu = 2 * W + 2;
  const long total = (long)(2 * h + 2) * Wu * B * cv;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const int v = (int)(i % cv);
    const long cell = i / cv;                             // (Y * Wu + X) * B + b
    const int b = (int)(cell % B);
    const long pix = cell / B;
    const int Y = (int)(pix / Wu), X = (int)(pix % Wu);
    uint4 val = make_uint4(0, 0, 0, 0);
    if (X != 0 && X != Wu - 1) {
      const int py = Y == 0 ? 0 : (Y == 2 * h + 1 ? h + 1 : 1 + (Y - 1) / 2);
      const int px = 1 + (X - 1) / 2;
      val = reinterpret_cast<const uint4 *>(P + (((long)py * (W + 2) + px) * B + b) * C)[v];
    }
    reinterpret_cast<uint4 *>(U + cell * C)[v] = val;
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
                        unsigned *ticket, cudaStream_t s, double *out2, double *out3) {
  if (B > 2 || B < 1 || C % 4 || C % GN_G || C > 4 * GNP_THREADS * 3 || !ws || !ticket ||
      M > (1L << 30))
    return cudaErrorInvalidValue;
  static_assert(GNP_SETROW0 + GNP_MAXB / GNP_SET + 1 <= GN_PARTIAL_BLOCKS, "workspace rows");
  if (M == 0) {
    for (double *o : {out, out2, out3})
      if (o) {
        const cudaError_t e = cudaMemsetAsync(o, 0, (size_t)B * GN_G * 2 * sizeof(double), s);
        if (e != cudaSuccess) return e;
      }
    return cudaSuccess;
  }
  // >= 8 rows per thread slot when the band allows, <= GNP_MAXB blocks
  const int nvec = C / 4, slots = nvec >= GNP_THREADS ? 1 : GNP_THREADS / nvec;
  const int nv = (nvec + GNP_THREADS - 1) / GNP_THREADS;
  const long rows_min = 8L * slots;
  long nb = std::max<long>(1, std::min<long>((M + rows_min - 1) / rows_min, GNP_MAXB));
  int rpb = (int)((M + nb - 1) / nb);
  rpb += rpb & 1;  // even: the batch index of a row is its parity (B = 2)
  nb = (M + rpb - 1) / rpb;
  const size_t smem = (size_t)2 * slots * B * C * sizeof(float);
  cudaError_t el;
  if (nv <= 1)
    el = launch_pdl(gn_partials_kernel<1>, dim3((unsigned)nb), dim3(GNP_THREADS), smem, s, x,
                    (int)M, B, C, rpb, ws, ticket, out, out2, out3);
  else if (nv == 2)
    el = launch_pdl(gn_partials_kernel<2>, dim3((unsigned)nb), dim3(GNP_THREADS), smem, s, x,
                    (int)M, B, C, rpb, ws, ticket, out, out2, out3);
  else
    el = launch_pdl(gn_partials_kernel<3>, dim3((unsigned)nb), dim3(GNP_THREADS), smem, s, x,
                    (int)M, B, C, rpb, ws, ticket, out, out2, out3);
  ++g_launches;
  return el;
}

template <typename T>
cudaError_t gn_apply(const float *x, int h, int W, int B, int C, const double *stats, int G,
                     double n_total, const float *gamma, const float *beta, float eps, int act,
                     int pad, T *out, cudaStream_t s, int zero_halo) {
  if (C % 4 || (stats && C % GN_G) || B > 2 || (long)h * W * B * (C / 4) > (1L << 30))
    return cudaErrorInvalidValue;
  const long M = (long)h * W * B;
  if (M == 0) return cudaSuccess;
  // ~GNA_UNR float4 per thread per block, <= 4 blocks per SM; rpb even (B = 2 pairs)
  const long vec = M * (C / 4);
  long nb = std::max<long>(1, std::min<long>(vec / (GNA_UNR * GNA_THREADS), 148L * 4));
  int rpb = (int)((M + nb - 1) / nb);
  rpb += rpb & 1;
  nb = (M + rpb - 1) / rpb;
  const size_t smem = stats ? (size_t)(2 * B + 1) * C * sizeof(float) : 0;
  if (smem > 48 * 1024) {
    static bool attr = false;
    if (!attr) {
      const cudaError_t e = cudaFuncSetAttribute(
          gn_apply_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      if (e != cudaSuccess) return e;
      attr = true;
    }
  }
  const cudaError_t el =
      launch_pdl(gn_apply_kernel<T>, dim3((unsigned)nb), dim3(GNA_THREADS), smem, s, x, h, W, B,
                 C, rpb, stats, G, n_total, gamma, beta, eps, act, pad, out, zero_halo);
  ++g_launches;
  return el;
}
template cudaError_t gn_apply<bf16>(const float *, int, int, int, int, const double *, int,
                                    double, const float *, const float *, float, int, int, bf16 *,
                                    cudaStream_t, int);
template cudaError_t gn_apply<float>(const float *, int, int, int, int, const double *, int,
                                     double, const float *, const float *, float, int, int,
                                     float *, cudaStream_t, int);

template <typename T>
cudaError_t upsample_pad(const T *P, int h, int W, int B, int C, T *U, cudaStream_t s) {
  if ((C * sizeof(T)) % 16) return cudaErrorInvalidValue;
  const long work = (long)(2 * h + 2) * (2 * W + 2) * B * (C * sizeof(T) / 16);
  const cudaError_t el = launch_pdl(upsample_pad_kernel<T>, dim3(grid_for(work)), dim3(256), 0, s,
                                    P, h, W, B, C, U);
  ++g_launches;
  return el;
}
template cudaError_t upsample_pad<bf16>(const bf16 *, int, int, int, int, bf16 *, cudaStream_t);
template cudaError_t upsample_pad<float>(const float *, int, int, int, int, float *, cudaStream_t);

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
cudaError_t latent_pad(const float *x, int h, int W, int Cl, int B, T *out, cudaStream_t s,
                       int zero_halo) {
  const long work = (long)(h + 2) * (W + 2) * B * Cl;
  const cudaError_t el = launch_pdl(latent_pad_kernel<T>, dim3(grid_for(work)), dim3(256), 0, s, x,
                                    h, W, Cl, B, out, zero_halo);
  ++g_launches;
  return el;
}
template cudaError_t latent_pad<bf16>(const float *, int, int, int, int, bf16 *, cudaStream_t,
                                      int);
template cudaError_t latent_pad<float>(const float *, int, int, int, int, float *, cudaStream_t,
                                       int);

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
