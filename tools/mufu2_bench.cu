// Microbenchmark: element throughput of MUFU ex2 variants (f32, f16x2, bf16x2)
// and whether the bf16x2 pack (F2FP) shares the MUFU / XU pipe with ex2.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
__global__ void ex2_f32(float *out, int iters) {
  float a = threadIdx.x * 1e-3f, b = a + 0.5f, c = a + 0.25f, d = a + 0.125f;
  long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
  }
  long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[0] += a + b + c + d;
}
__global__ void ex2_f16x2(float *out, int iters) {
  unsigned a = 0x3c003c00u + threadIdx.x, b = a ^ 1, c = a ^ 2, d = a ^ 3;
  long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a));
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(b));
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(c));
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(d));
  }
  long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[0] += (float)(a ^ b ^ c ^ d);
}
__global__ void ex2_bf16x2(float *out, int iters) {
  unsigned a = 0x3f803f80u + threadIdx.x, b = a ^ 1, c = a ^ 2, d = a ^ 3;
  long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a));
    asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(b));
    asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(c));
    asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(d));
  }
  long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[0] += (float)(a ^ b ^ c ^ d);
}
// 4 ex2.f32 + 2 bf16x2 packs per iteration (the softmax mix)
__global__ void ex2_pack(float *out, int iters) {
  float a = threadIdx.x * 1e-3f, b = a + 0.5f, c = a + 0.25f, d = a + 0.125f;
  unsigned r = 0;
  long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
    unsigned u, v;
    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(a), "f"(b));
    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(v) : "f"(c), "f"(d));
    r ^= u ^ v;
  }
  long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[0] += r;
}
// 4 ex2.f32 + 2 integer (round-half-up) bf16x2 packs per iteration
__global__ void ex2_ipack(float *out, int iters) {
  float a = threadIdx.x * 1e-3f, b = a + 0.5f, c = a + 0.25f, d = a + 0.125f;
  unsigned r = 0;
  long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
    unsigned u = __byte_perm(__float_as_uint(a) + 0x8000u, __float_as_uint(b) + 0x8000u, 0x7632);
    unsigned v = __byte_perm(__float_as_uint(c) + 0x8000u, __float_as_uint(d) + 0x8000u, 0x7632);
    r ^= u ^ v;
  }
  long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[0] += r;
}
// packs only (F2FP), 2 per iteration, independent inputs
__global__ void pack_only(float *out, int iters) {
  float a = threadIdx.x * 1e-3f, b = a + 0.5f, c = a + 0.25f, d = a + 0.125f;
  unsigned r = 0;
  long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    unsigned u, v;
    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(a), "f"(b));
    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(v) : "f"(c), "f"(d));
    r ^= u ^ v;
    a = __uint_as_float(__float_as_uint(a) ^ (r & 1));
  }
  long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[0] += r;
}
// f16x2 path per pair: cvt f32x2->f16x2, ex2.f16x2, unpack to f32 (2 cvt), pack bf16x2
__global__ void f16_path(float *out, int iters) {
  float a = threadIdx.x * -1e-3f, b = a - 0.5f, c = a - 0.25f, d = a - 0.125f;
  unsigned r = 0;
  float s = 0.f;
  long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    unsigned h0, h1;
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h0) : "f"(a), "f"(b));
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h1) : "f"(c), "f"(d));
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h0));
    asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h1));
    __half2 x0 = *reinterpret_cast<__half2 *>(&h0), x1 = *reinterpret_cast<__half2 *>(&h1);
    float2 f0 = __half22float2(x0), f1 = __half22float2(x1);
    unsigned u, v;
    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(f0.x), "f"(f0.y));
    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(v) : "f"(f1.x), "f"(f1.y));
    r ^= u ^ v;
    s += f0.x + f0.y + f1.x + f1.y;
    a -= 1e-3f; b -= 1e-3f; c -= 1e-3f; d -= 1e-3f;
  }
  long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[0] += r + s;
}
int main() {
  float *d; cudaMalloc(&d, 8); float h[2];
  const int iters = 4096;
  for (int threads : {256, 512, 1024}) {
#define RUN(k, per)                                                                   \
    k<<<148, threads>>>(d, iters); cudaDeviceSynchronize();                           \
    k<<<148, threads>>>(d, iters); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);       \
    printf("%-10s threads/SM %4d: %.2f elem/clk/SM\n", #k, threads, (per) * iters * threads / h[1]);
    RUN(ex2_f32, 4.0)
    RUN(ex2_f16x2, 8.0)
    RUN(ex2_bf16x2, 8.0)
    RUN(ex2_pack, 4.0)
    RUN(f16_path, 4.0)
    RUN(ex2_ipack, 4.0)
    RUN(pack_only, 4.0)
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
