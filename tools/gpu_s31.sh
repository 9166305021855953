# GEMM epilogue warps 8 (168 regs, spills) vs 4 (239 regs, no spills): kbench A/B + GEMM parity
mkdir -p gpurun_out
d=paper_2509_04719_b200/csrc/kernels
for v in "-DSTADI_GEMM_EPI_WARPS=4" base "-DSTADI_GEMM_EPI_WARPS=4" base; do
  defs=""; [ "$v" != base ] && defs="$v"
  touch $d/tc_gemm.cu; STADI_NVCC_EXTRA="$defs" python -m paper_2509_04719_b200.build > /tmp/b.log 2>&1 || { echo "build failed $v"; tail -3 /tmp/b.log; }
  echo "== $v"
  timeout 300 python tools/kbench.py gemm 2>&1 | grep gemm
  timeout 300 python tools/kbench.py conv 2>&1 | grep conv3x3
done | tee gpurun_out/s31_ab.txt
touch $d/tc_gemm.cu; STADI_NVCC_EXTRA="-DSTADI_GEMM_EPI_WARPS=4" python -m paper_2509_04719_b200.build > /tmp/b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "gemm or conv" -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/s31_tests.log 2>&1
echo "pytest (EPI_WARPS=4) rc=$?"; tail -2 gpurun_out/s31_tests.log
