# residual-RMW epilogue loads one chunk ahead: same-box A/B vs HEAD, and the env switch
mkdir -p gpurun_out
bash tools/gpu_src_ab.sh tc_gemm.cu tools/ab_tc_gemm_head.cu gemm "epi=2|epi=3|epi=5" 2>&1 | tee gpurun_out/s19_ab.txt
for v in 0 1; do echo "== RES_PIPE=$v"; STADI_RES_PIPE=$v timeout 300 python tools/kbench.py gemm 2>&1 | grep -E "epi=2|epi=3"; done | tee -a gpurun_out/s19_ab.txt
timeout 300 python tools/kbench.py conv 2>&1 | grep conv3x3 | tee -a gpurun_out/s19_ab.txt
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "gemm or conv" -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/s19_tests.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/s19_tests.log
