// Microbenchmark: does a resident "occupancy" kernel slow unrelated small kernels
// on the free SMs?  Variants of the resident kernel: 0 none, 1 sleep + poll host
// flag (thread 0) + barrier, 2 sleep + poll DEVICE flag, 3 barrier only (thread 0
// sleeps without polling until a device flag), 4 FMA spin.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void resident(volatile int *host_stop, volatile int *dev_stop, int mode, int iters) {
  extern __shared__ float pad[];
  if (threadIdx.x == 0) {
    if (mode == 1) while (!*host_stop) __nanosleep(20000);
    else if (mode == 2 || mode == 3) while (!*dev_stop) __nanosleep(mode == 2 ? 20000 : 1000000);
    pad[0] = 0.f;
  }
  if (mode == 4) {
    float a = threadIdx.x;
    while (!*dev_stop) for (int k = 0; k < 4096; ++k) a = fmaf(a, 1.0001f, 1e-7f);
    if (a == 1.f) pad[1] = a;
  }
  __syncthreads();
}
__global__ void tiny(float *x, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 0.999f + 1e-3f;
}
int main() {
  int *hs, *ds;
  cudaHostAlloc(&hs, 4, cudaHostAllocMapped);
  cudaMalloc(&ds, 4);
  int *hs_dev;
  cudaHostGetDevicePointer(&hs_dev, hs, 0);
  float *x;
  cudaMalloc(&x, 1 << 24);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  int smem = 0;
  cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaFuncSetAttribute(resident, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode <= 4; ++mode) {
    for (int nres : {30, 60}) {
      *hs = 0;
      cudaMemset(ds, 0, 4);
      cudaDeviceSynchronize();
      if (mode) resident<<<nres, 1024, smem, s1>>>(hs_dev, ds, mode, 0);
      for (int n : {16384, 1 << 22}) {
        for (int w = 0; w < 20; ++w) tiny<<<(n + 255) / 256, 256, 0, s2>>>(x, n);
        cudaEventRecord(e0, s2);
        for (int w = 0; w < 200; ++w) tiny<<<(n + 255) / 256, 256, 0, s2>>>(x, n);
        cudaEventRecord(e1, s2);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("mode %d resident CTAs %d  n=%8d: %.2f us per tiny kernel\n", mode, mode ? nres : 0, n,
               ms * 1000 / 200);
      }
      *hs = 1;
      int one = 1;
      cudaMemcpyAsync(ds, &one, 4, cudaMemcpyHostToDevice, s2);
      cudaDeviceSynchronize();
      if (!mode) break;
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
