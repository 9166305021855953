# P-over-S attention with larger key tiles: parity + C5-shape microbench per STADI_ATTN_AKT.
# Usage: bash tools/gpu_attn_akt.sh <tag>
tag=${1:-x}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "alias" -q -p no:cacheprovider \
  > gpurun_out/akt_tests_$tag.log 2>&1; echo "tests rc=$?"; tail -n 3 gpurun_out/akt_tests_$tag.log
for v in "STADI_ATTN_ALIAS=0" ${VARIANTS:-"STADI_ATTN_ALIAS=1,STADI_ATTN_AKT=0" "STADI_ATTN_ALIAS=1,STADI_ATTN_AKT=144" "STADI_ATTN_ALIAS=1,STADI_ATTN_AKT=160" "STADI_ATTN_ALIAS=1,STADI_ATTN_AKT=176" "STADI_ATTN_ALIAS=1,STADI_ATTN_AKT=177" "STADI_ATTN_ALIAS=1,STADI_ATTN_AKT=178" "STADI_ATTN_ALIAS=1,STADI_ATTN_AKT=161"}; do
  echo "== $v"; for i in 1 2; do env ${v//,/ } timeout 120 python tools/kbench.py attn 2>&1 | grep "hd=72"; done
done
