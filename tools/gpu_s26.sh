# residual-epilogue switches A/B (L2 prefetch, 16-byte RMW) on the fp32-residual GEMM shapes
mkdir -p gpurun_out
for v in "X=1" "STADI_RES_PREFETCH=0" "X=1" "STADI_RES_PREFETCH=0"; do
  echo "== $v"; env $v timeout 300 python tools/kbench.py gemm 2>&1 | grep -E "epi=2|epi=3"
  env $v timeout 300 python tools/kbench.py conv 2>&1 | grep "conv3x3"
done | tee gpurun_out/s26_ab.txt
