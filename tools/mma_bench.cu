// Microbenchmark: tcgen05.mma kind::f16 issue/execute rate vs N (M = 128, K = 16),
// SS form (A, B in smem) and TS form (A in TMEM).  One CTA per SM.
#include <cstdio>
#include "device.cuh"
using namespace stadi;
template <int N, bool TS>
__global__ void mma_loop(float *out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = umma_idesc_bf16(128, N, 0, 0);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const uint64_t ad = umma_desc(a, 16, 1024, SWZ_128B), bd = umma_desc(b, 16, 1024, SWZ_128B);
    long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if constexpr (TS) umma_bf16_ts(tmem, tmem + 256, bd, id, 1);
      else umma_bf16(tmem, ad, bd, id, 1);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (float)(t1 - t0) / iters;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(slot, 512); }
}
template <int N, bool TS>
void run(float *d) {
  float h;
  cudaFuncSetAttribute(mma_loop<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  mma_loop<N, TS><<<148, 128, 65536>>>(d, 4096);
  mma_loop<N, TS><<<148, 128, 65536>>>(d, 4096);
  cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  printf("%s N=%3d: %.1f clk per MMA (floor %d)  %s\n", TS ? "TS" : "SS", N, h, 128 * N / 256,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  float *d; cudaMalloc(&d, 8);
  run<16, false>(d); run<32, false>(d); run<16, true>(d); run<32, true>(d);
  run<64, false>(d); run<80, false>(d); run<112, false>(d); run<128, false>(d); run<256, false>(d);
  run<64, true>(d); run<80, true>(d); run<128, true>(d); run<256, true>(d);
}
