# Attention experiment: tests, C5-shaped microbench A/B over $VARIANTS, CTA-0 timelines.
# Usage: bash tools/gpu_attn_exp.sh <tag>
tag=${1:-x}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -k attention -q -x -p no:cacheprovider \
  > gpurun_out/attn_tests_$tag.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/attn_tests_$tag.log
for v in ${VARIANTS:-STADI_ATTN_DEFER=0 STADI_ATTN_DEFER=1}; do
  echo "== $v"; for i in 1 2; do env ${v//,/ } timeout 120 python tools/kbench.py attn 2>&1 | grep "hd=72"; done
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -rdc=true -DSTADI_ATTN_TRACE \
  -Iinclude -Ipaper_2509_04719_b200/csrc tools/attn_trace.cu \
  paper_2509_04719_b200/csrc/kernels/{tc_attn,tc_gemm,simt}.cu -lcuda -o /tmp/attn_trace 2>&1 | grep -i error
for v in ${TRACE_VARIANTS:-STADI_ATTN_DEFER=0 STADI_ATTN_DEFER=1}; do
  echo "== trace $v"; env ${v//,/ } timeout 60 /tmp/attn_trace 72 | sed -n '9,20p'
done
