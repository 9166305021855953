# GEMM A/B: parity of the GEMM / conv kernels (split-K included), then the GEMM
# microbench per pair mode and with split-K off.  Usage: bash tools/gpu_gemm_ab.sh [tag]
tag=${1:-ab}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "gemm or conv" -q -x \
  -p no:cacheprovider > gpurun_out/gemm_tests_$tag.log 2>&1
echo "kernel tests rc=$?"; tail -n 2 gpurun_out/gemm_tests_$tag.log
for v in ${VARIANTS:-STADI_GEMM_MC=dflt STADI_SPLITK=0}; do
  echo "== $v"; env $v timeout 300 python tools/kbench.py gemm 2>&1 | grep -i "gemm\|error"
done
