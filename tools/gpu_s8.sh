# round-2 session-3 evidence: GPU tests, C5 / C4 bench lines, C5 launch list, ncu --set full of
# the attention and the largest GEMM
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rfE > gpurun_out/s8_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/s8_tests.log
timeout 900 python bench.py > gpurun_out/bench_c5_s8.json 2> gpurun_out/bench_c5_s8.err
python -c "import json; d=json.load(open('gpurun_out/bench_c5_s8.json')); print('c5', d['ms_per_step'], d['clocks'], d['roofline']['achieved'], d['roofline']['frac'], {k:(v['launches'], round(v['ms']/d['steps'],1), v['tflops']) for k,v in d['kernels'].items()})"
timeout 900 python bench.py --workload c4 > gpurun_out/bench_c4_s8.json 2> gpurun_out/bench_c4_s8.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_s8.json')); print('c4', d['ms_per_step'], d['clocks'], {k:(v['launches'], round(v['ms']/d['steps'],1), v['tflops']) for k,v in d['kernels'].items()})"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 22000 -c 6000 --csv \
  --log-file gpurun_out/s8_c5_launches.csv python bench.py --steps 1 --warmup 3 --ncu > gpurun_out/s8_ncu_list.log 2>&1
echo "list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -s 200 -c 1 \
  -o gpurun_out/s8_attn python bench.py --steps 1 --warmup 3 --ncu > gpurun_out/s8_ncu_attn.log 2>&1
echo "attn rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 400 -c 1 \
  -o gpurun_out/s8_gemm python bench.py --steps 1 --warmup 3 --ncu > gpurun_out/s8_ncu_gemm.log 2>&1
echo "gemm rc=$?"
