# Build + run the attention timeline trace for $TRACE_VARIANTS (each may carry NVCCDEF=...).
for v in ${TRACE_VARIANTS:-base}; do
  defs=""; envs=""
  for kv in ${v//,/ }; do case $kv in -D*) defs="$defs $kv";; base) ;; *) envs="$envs $kv";; esac; done
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -rdc=true -DSTADI_ATTN_TRACE $defs \
    -Iinclude -Ipaper_2509_04719_b200/csrc tools/attn_trace.cu \
    paper_2509_04719_b200/csrc/kernels/{tc_attn,tc_gemm,simt}.cu -lcuda -o /tmp/attn_trace 2>&1 | grep -i error
  echo "== trace $v"; env $envs timeout 60 /tmp/attn_trace 72 | sed -n '9,14p'
done
