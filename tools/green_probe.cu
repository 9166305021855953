// Probe: CUDA green contexts (SM partitions) on B200 driven from the runtime API.
// Two partitions; a kernel launched with <<<>>> into each partition's stream records
// the SMs its CTAs ran on and spins; checks (1) disjoint SM sets of the right size,
// (2) concurrency (both partitions busy at once), (3) primary-context cudaMalloc
// memory is usable from green-context kernels.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/green_probe.cu -lcuda -o /tmp/green_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <set>
#define CKD(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)
#define CKR(x) do { cudaError_t r = (x); if (r != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(r)); return 1; } } while (0)

__global__ void spin(int *smids, long long cycles) {
  unsigned sm;
  asm("mov.u32 %0, %%smid;" : "=r"(sm));
  if (threadIdx.x == 0) smids[blockIdx.x] = (int)sm;
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}

int main(int argc, char **argv) {
  int a = argc > 1 ? atoi(argv[1]) : 72, b = argc > 2 ? atoi(argv[2]) : 72;
  CKR(cudaSetDevice(0));
  CKR(cudaFree(0));
  CUdevice dev; CKD(cuDeviceGet(&dev, 0));
  CUdevResource all; CKD(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", all.sm.smCount);
  // split into groups of 8 SMs (the sm_90+ granularity), then give each partition
  // a/8 resp. b/8 of the groups
  CUdevResource grp[32], rest; unsigned n = 32;
  CKD(cuDevSmResourceSplitByCount(grp, &n, &all, &rest, 0, 8));
  printf("groups: %u of %u SMs (rest %u)\n", n, grp[0].sm.smCount, rest.sm.smCount);
  const int na = a / 8, nbg = b / 8;
  if (na + nbg > (int)n) { printf("FAIL not enough groups\n"); return 1; }
  CUdevResourceDesc da, db; CKD(cuDevResourceGenerateDesc(&da, grp, na)); CKD(cuDevResourceGenerateDesc(&db, grp + na, nbg));
  CUdevResource ga = grp[0], gb = grp[na]; ga.sm.smCount = 8 * na; gb.sm.smCount = 8 * nbg;
  printf("partitions: %u + %u\n", ga.sm.smCount, gb.sm.smCount);
  CUgreenCtx gca, gcb; CKD(cuGreenCtxCreate(&gca, da, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CKD(cuGreenCtxCreate(&gcb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sa, sb; CKD(cuGreenCtxStreamCreate(&sa, gca, CU_STREAM_NON_BLOCKING, 0));
  CKD(cuGreenCtxStreamCreate(&sb, gcb, CU_STREAM_NON_BLOCKING, 0));
  int *ia, *ib; const int nb = 148 * 4;
  CKR(cudaMalloc(&ia, nb * 4)); CKR(cudaMalloc(&ib, nb * 4));   // primary context memory
  const long long cyc = 2000000;
  cudaEvent_t e0, e1; CKR(cudaEventCreate(&e0)); CKR(cudaEventCreate(&e1));
  // serial reference on the primary context: one partition-sized grid
  CKR(cudaEventRecord(e0, 0));
  spin<<<nb, 128, 0, 0>>>(ia, cyc);
  CKR(cudaEventRecord(e1, 0)); CKR(cudaEventSynchronize(e1));
  float ms_full; cudaEventElapsedTime(&ms_full, e0, e1);
  // both partitions at once
  CKR(cudaEventRecord(e0, 0));
  CKR(cudaStreamWaitEvent((cudaStream_t)sa, e0, 0)); CKR(cudaStreamWaitEvent((cudaStream_t)sb, e0, 0));
  spin<<<nb, 128, 0, (cudaStream_t)sa>>>(ia, cyc);
  CKR(cudaGetLastError());
  spin<<<nb, 128, 0, (cudaStream_t)sb>>>(ib, cyc);
  CKR(cudaGetLastError());
  cudaEvent_t ea, eb; CKR(cudaEventCreate(&ea)); CKR(cudaEventCreate(&eb));
  CKR(cudaEventRecord(ea, (cudaStream_t)sa)); CKR(cudaEventRecord(eb, (cudaStream_t)sb));
  CKR(cudaStreamWaitEvent(0, ea, 0)); CKR(cudaStreamWaitEvent(0, eb, 0));
  CKR(cudaEventRecord(e1, 0)); CKR(cudaEventSynchronize(e1));
  float ms_two; cudaEventElapsedTime(&ms_two, e0, e1);
  std::vector<int> ha(nb), hb(nb);
  CKR(cudaMemcpy(ha.data(), ia, nb * 4, cudaMemcpyDeviceToHost));
  CKR(cudaMemcpy(hb.data(), ib, nb * 4, cudaMemcpyDeviceToHost));
  std::set<int> sa_(ha.begin(), ha.end()), sb_(hb.begin(), hb.end());
  int inter = 0; for (int x : sa_) inter += sb_.count(x);
  printf("full-GPU grid %.2f ms; two partitions concurrently %.2f ms (serial would be ~%.2f x 2 x 148/%u)\n",
         ms_full, ms_two, ms_full, ga.sm.smCount);
  printf("SMs used: A %zu, B %zu, overlap %d\n", sa_.size(), sb_.size(), inter);
  return 0;
}
