# GEMM pair-mode A/B: parity of the GEMM / conv kernels with the cta_group::2 mode,
# then the C5-shaped GEMM microbench per mode.  Usage: bash tools/gpu_gemm_ab.sh [tag]
tag=${1:-ab}
mkdir -p gpurun_out
for m in 3 2; do
  STADI_GEMM_MC=$m timeout 600 python -m pytest tests/test_gpu_kernels.py -k "gemm or conv" -q -x \
    -p no:cacheprovider > gpurun_out/gemm_tests_mc${m}_$tag.log 2>&1
  echo "MC=$m kernel tests rc=$?"; tail -n 2 gpurun_out/gemm_tests_mc${m}_$tag.log
done
for m in 2 3 0; do
  echo "== STADI_GEMM_MC=$m"; STADI_GEMM_MC=$m timeout 300 python tools/kbench.py gemm 2>&1 | grep -i "gemm\|error"
done
