# hd-40 attention: narrow 3 x 16 chunks (one N = 48 PV MMA per 16 keys) A/B + parity
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -k "alias_variant" -m gpu -q -p no:cacheprovider > gpurun_out/s22_tests.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/s22_tests.log
for v in 0 1 0 1; do echo "== NARROW40=$v"; STADI_ATTN_NARROW40=$v timeout 120 python tools/kbench.py attn 2>&1 | grep "hd=40"; STADI_ATTN_NARROW40=$v timeout 120 python tools/kbench.py xattn 2>&1 | grep "hd=40"; done | tee gpurun_out/s22_ab.txt
Q="--no-method --no-occ-sweep --no-cpu-baseline --no-uniform --no-e2e"
for v in 0 1; do
  STADI_ATTN_NARROW40=$v timeout 900 python bench.py --workload c3 $Q > gpurun_out/bench_c3_s22_$v.json 2> gpurun_out/bench_c3_s22_$v.err
  python -c "import json; d=json.load(open('gpurun_out/bench_c3_s22_$v.json')); print('c3 NARROW40=$v', d['ms_per_step'], {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"
done
