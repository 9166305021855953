# S read in two halves (STADI_ATTN_SPLITLD) A/B + attention parity
mkdir -p gpurun_out
BUILD_VARIANTS="-DSTADI_ATTN_SPLITLD=0 base -DSTADI_ATTN_SPLITLD=0 base" bash tools/gpu_attn_build_ab.sh 2>&1 | tee gpurun_out/s15_ab.txt
timeout 300 python tools/kbench.py attn 2>&1 | tee -a gpurun_out/s15_ab.txt
