# two-CTAs-per-SM attention variant for mid-length K/V (STADI_ATTN_DUAL_KV) A/B
mkdir -p gpurun_out
for v in 256 1024 4096 256 1024; do echo "== DUAL_KV=$v"; STADI_ATTN_DUAL_KV=$v timeout 120 python tools/kbench.py small 2>&1; done | tee gpurun_out/s21_dual_ab.txt
Q="--no-method --no-occ-sweep --no-cpu-baseline --no-uniform --no-e2e"
for wl in c3 c4; do for v in 256 1024; do
  STADI_ATTN_DUAL_KV=$v timeout 900 python bench.py --workload $wl $Q > gpurun_out/bench_${wl}_s21_$v.json 2> gpurun_out/bench_${wl}_s21_$v.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${wl}_s21_$v.json')); print('$wl DUAL_KV=$v', d['ms_per_step'], {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"
done; done
