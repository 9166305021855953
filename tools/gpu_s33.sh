# implicit conv tile width A/B (STADI_GEMM_BN; split-K off when forced)
mkdir -p gpurun_out
for v in 0 64 0 64; do echo "== BN=$v"; STADI_GEMM_BN=$v timeout 300 python tools/kbench.py conv 2>&1 | grep conv3x3; STADI_GEMM_BN=$v timeout 300 python tools/kbench.py unet 2>&1 | grep "mode=1 implicit=1\|mode=2 implicit=1"; done | tee gpurun_out/s33_conv_bn_ab.txt
