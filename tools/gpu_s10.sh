# single-tile P-over-S cross-attention A/B, attention tests, C5 bench + launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "attention" -m gpu -q -p no:cacheprovider --timeout 300 -rfE > gpurun_out/s10_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/s10_tests.log
for v in 0 1 0 1; do echo "== XTILE=$v"; STADI_ATTN_XTILE=$v timeout 120 python tools/kbench.py xattn 2>&1; done | tee gpurun_out/s10_xattn_ab.txt
for v in 0 1 0 1; do echo "== SPEC=$v"; STADI_ATTN_SPEC=$v timeout 120 python tools/kbench.py attn 2>&1; done | tee gpurun_out/s10_spec_ab.txt
timeout 900 python bench.py > gpurun_out/bench_c5_s10.json 2> gpurun_out/bench_c5_s10.err
python -c "import json; d=json.load(open('gpurun_out/bench_c5_s10.json')); print('c5', d['ms_per_step'], d['clocks'], d['roofline']['achieved'], d['roofline']['frac'], {k:(v['launches'], round(v['ms']/d['steps'],1), v['tflops']) for k,v in d['kernels'].items()})"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 4000 -c 6400 --csv \
  --log-file gpurun_out/s10_c5_launches.csv python bench.py --steps 1 --warmup 3 --ncu > gpurun_out/s10_ncu_list.log 2>&1
echo "list rc=$?"; grep -c gpu__time gpurun_out/s10_c5_launches.csv
