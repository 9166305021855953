# A/B of compile-time attention variants through the kernel-level ABI: rebuilds
# libstadi.so with each NVCC define set in $BUILD_VARIANTS (space separated; a
# variant is comma-separated -D defines or "base"), runs the attention tests once
# and the C5-shaped microbench 2x per variant.  $ATTN_ENV: run-time switches.
for v in ${BUILD_VARIANTS:-base}; do
  defs=""; for kv in ${v//,/ }; do case $kv in -D*) defs="$defs $kv";; esac; done
  STADI_NVCC_EXTRA="$defs" python -m paper_2509_04719_b200.build > /tmp/build.log 2>&1 || { echo "build failed $v"; tail -5 /tmp/build.log; continue; }
  echo "== $v"
  case "$v" in *NO*) ;; *) env $ATTN_ENV timeout 300 python -m pytest tests/test_gpu_kernels.py -k attention -q -x -p no:cacheprovider 2>&1 | tail -1;; esac
  for i in 1 2; do env $ATTN_ENV timeout 120 python tools/kbench.py attn 2>&1 | grep "hd=72"; done
  touch paper_2509_04719_b200/csrc/kernels/tc_attn.cu
done
