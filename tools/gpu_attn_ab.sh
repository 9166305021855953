# Attention A/B on the GPU: parity tests of both softmax layouts, then the C5-shaped
# microbench for the variants in $VARIANTS (env assignments separated by spaces,
# commas inside one variant).  Usage: bash tools/gpu_attn_ab.sh [tag]
tag=${1:-ab}
mkdir -p gpurun_out
for qd in 1 0; do
  STADI_ATTN_QUAD=$qd timeout 600 python -m pytest tests/test_gpu_kernels.py -k attention -q -x \
    -p no:cacheprovider > gpurun_out/attn_tests_q${qd}_$tag.log 2>&1
  echo "QUAD=$qd tests rc=$?"; tail -n 2 gpurun_out/attn_tests_q${qd}_$tag.log
done
for v in ${VARIANTS:-STADI_ATTN_QUAD=0 STADI_ATTN_QUAD=1 STADI_ATTN_TOK=0 STADI_ATTN_POLY=1}; do
  echo "== $v"; env ${v//,/ } timeout 120 python tools/kbench.py attn 2>&1 | grep attn
done
