# DUAL40 default on: GPU suite + C3 bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rfE > gpurun_out/s24_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/s24_tests.log
timeout 900 python bench.py --workload c3 > gpurun_out/bench_c3_s24.json 2> gpurun_out/bench_c3_s24.err
python -c "import json; d=json.load(open('gpurun_out/bench_c3_s24.json')); print('c3', d['ms_per_step'], d['clocks']['sm_mhz'], d['path_roofline']['frac'], {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"
