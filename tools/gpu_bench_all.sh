# Bench lines of every workload at N = 1.  Usage: bash tools/gpu_bench_all.sh <tag>
tag=${1:-r}
mkdir -p gpurun_out
for wl in c5 c4 c3 c2; do
  timeout 1200 python bench.py --workload $wl > gpurun_out/bench_${wl}_$tag.json 2> gpurun_out/bench_${wl}_$tag.err
  echo "$wl rc=$?"; tail -2 gpurun_out/bench_${wl}_$tag.err
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_${wl}_$tag.json')); print(d['config']['workload'][:40], 'ms/img', round(d['ms_per_step'],1), 'roof', d['roofline']['class'], round(d['roofline']['frac'],3), {k: (round(v['tflops']) if v['tflops'] else None) for k,v in d['kernels'].items()})"
done
