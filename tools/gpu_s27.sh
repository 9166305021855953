# final HEAD check: smoke + the default bench line
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_c5_s27.json 2> gpurun_out/bench_c5_s27.err
echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c5_s27.json')); print('c5', d['ms_per_step'], d['clocks'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'])"
