# GEMM planner L2 default on C5 / C2 (quick bench legs), then the full GPU suite
mkdir -p gpurun_out
Q="--no-method --no-occ-sweep --no-cpu-baseline --no-uniform --no-e2e"
for wl in c2 c5; do for l2 in 6300 12600; do
  STADI_GEMM_L2=$l2 timeout 900 python bench.py --workload $wl $Q > gpurun_out/bench_${wl}_s13_$l2.json 2> gpurun_out/bench_${wl}_s13_$l2.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${wl}_s13_$l2.json')); print('$wl L2=$l2', d['ms_per_step'], d['clocks'], {k:(v['launches'], round(v['ms']/d['steps'],1), v['tflops']) for k,v in d['kernels'].items()})"
done; done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rfE > gpurun_out/s13_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/s13_tests.log
