# GEMM CTA-pair mode A/B after the warp-collective MMA issuer (env STADI_GEMM_MC)
mkdir -p gpurun_out
for v in default 2 3 1; do
  echo "== MC=$v"
  if [ $v = default ]; then timeout 300 python tools/kbench.py gemm 2>&1 | grep gemm; timeout 300 python tools/kbench.py unet 2>&1 | grep -E "^gemm|^conv3x3 [0-9]";
  else STADI_GEMM_MC=$v timeout 300 python tools/kbench.py gemm 2>&1 | grep gemm; STADI_GEMM_MC=$v timeout 300 python tools/kbench.py unet 2>&1 | grep -E "^gemm|^conv3x3 [0-9]"; fi
done | tee gpurun_out/s20_mc_ab.txt
