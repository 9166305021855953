# final-state check: full GPU suite, smoke, the default bench line (all legs), attention kbench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rfE > gpurun_out/s17_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/s17_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 120 python tools/kbench.py attn 2>&1 | grep hd=72
timeout 1200 python bench.py > gpurun_out/bench_c5_s17.json 2> gpurun_out/bench_c5_s17.err
echo "bench rc=$?"; tail -2 gpurun_out/bench_c5_s17.err
python -c "import json; d=json.load(open('gpurun_out/bench_c5_s17.json')); print('c5', d['ms_per_step'], d['clocks'], d['roofline']['achieved'], d['roofline']['frac'], d['e2e'], (d.get('method_vgpu') or {}).get('stadi_latency_reduction'), d.get('cpu_baseline',{}).get('value'))"
