# fp32-residual GEMM tile width A/B (STADI_GEMM_BN) on the C5 out-projection shape
mkdir -p gpurun_out
for v in 0 64 128 192 0 64 128; do echo "== BN=$v"; STADI_GEMM_BN=$v timeout 300 python tools/kbench.py gemm 2>&1 | grep -E "N=1152 K=1152 epi=2|N=1152 K=4608"; done | tee gpurun_out/s28_bn_ab.txt
