// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM, by warps per CTA.
#include <cstdio>
#include "device.cuh"
using namespace stadi;
__global__ void tmem_ld_loop(float *out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0, r[32];
  long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    tmem_ld32_nowait(tmem + ((warp >> 2) * 64) % 512, r);
    tmem_ld32_nowait(tmem + ((warp >> 2) * 64 + 32) % 512, r);
    tmem_ld_wait();
    acc += r[i & 31];
  }
  long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  out[0] += acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(slot, 512);
  }
}
int main() {
  float *d; cudaMalloc(&d, 8); float h[2];
  const int iters = 2000;
  for (int warps : {4, 8, 16}) {
    tmem_ld_loop<<<148, warps * 32>>>(d, iters); cudaDeviceSynchronize();
    tmem_ld_loop<<<148, warps * 32>>>(d, iters); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)iters * warps * 32 * 64 * 4;
    printf("warps %2d: %.1f B/clk/SM  (%s)\n", warps, bytes / h[1], cudaGetErrorString(cudaGetLastError()));
  }
}
