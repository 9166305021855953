// Standalone timeline trace of the attention kernel (CTA 0): build on the box with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -rdc=true -DSTADI_ATTN_TRACE \
//     -Iinclude -Ipaper_2509_04719_b200/csrc tools/attn_trace.cu \
//     paper_2509_04719_b200/csrc/kernels/{tc_attn,tc_gemm,simt}.cu -o /tmp/attn_trace
#include <cstdio>
#include <vector>
#include "kernels.h"
namespace stadi { extern __device__ long long g_attn_trace[16 * 2 * 64]; }
using namespace stadi;
int main(int argc, char **argv) {
  const int Nq = 16384, Nkv = 16384, B = 2, hd = argc > 1 ? atoi(argv[1]) : 72, H = 1152 / hd;
  const size_t d = (size_t)H * hd;
  bf16 *q, *kv, *o;
  cudaMalloc(&q, Nq * B * d * 2); cudaMalloc(&kv, Nkv * B * 2 * d * 2); cudaMalloc(&o, Nq * B * d * 2);
  cudaMemset(q, 0, Nq * B * d * 2); cudaMemset(kv, 0, Nkv * B * 2 * d * 2);
  for (int i = 0; i < 3; ++i) tc_attention_bf16(q, kv, o, Nq, Nkv, B, H, hd, 0);
  cudaDeviceSynchronize();
  std::vector<long long> t(16 * 2 * 64);
  cudaMemcpyFromSymbol(t.data(), g_attn_trace, t.size() * 8);
  const char *names[15] = {"mma:s_free", "mma:S_iss", "mma:p_full", "sm:s_full",
                           "sm:loaded", "sm:max", "sm:p_arr", "sm:tok", "mma:PV_iss", "sm:o_done",
                           "sm:exp_end", "sm:pv_wait", "sm:st_done", "mma:top(g0)/pre_v(g1)",
                           "mma:k_full(g0)/v_full(g1)"};
  long long t0 = t[(3 * 2 + 0) * 64 + 0];
  for (int j = 0; j < 16; ++j)
    for (int g = 0; g < 2; ++g) {
      printf("j=%2d g=%d:", j, g);
      for (int e = 0; e < 15; ++e) printf(" %s=%6lld", names[e], t[(e * 2 + g) * 64 + j] - t0);
      printf("\n");
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
