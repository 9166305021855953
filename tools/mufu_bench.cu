// Microbenchmark: MUFU ex2 and F2FP throughput per SM (ops/clk).
#include <cstdio>
#include <cuda_bf16.h>
__global__ void ex2_loop(float *out, int iters) {
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
__global__ void cvt_loop(float *out, int iters) {
  float a = threadIdx.x * 1e-3f, b = a + 0.5f;
  unsigned r = 0;
  long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
    unsigned u = *reinterpret_cast<unsigned *>(&t);
    r ^= u;
    a += 1.f; b += 1.f;
  }
  long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[0] += r;
}
int main() {
  float *d; cudaMalloc(&d, 8); float h[2];
  const int iters = 4096;
  for (int threads : {128, 256, 512, 1024}) {
    ex2_loop<<<148, threads>>>(d, iters); cudaDeviceSynchronize();
    ex2_loop<<<148, threads>>>(d, iters); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("ex2: threads/SM %4d: %.2f ex2/clk/SM\n", threads, 4.0 * iters * threads / h[1]);
    cvt_loop<<<148, threads>>>(d, iters); cudaDeviceSynchronize();
    cvt_loop<<<148, threads>>>(d, iters); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("cvt: threads/SM %4d: %.2f loop-iter/clk/SM\n", threads, 1.0 * iters * threads / h[1]);
  }
}
