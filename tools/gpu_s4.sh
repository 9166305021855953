# session-3 round-2 measurement batch: GPU tests, U-Net kernel microbench, attention key-tile A/B,
# C3 bench line + launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rfE > gpurun_out/s4_tests.log 2>&1
echo "pytest rc=$?"; tail -8 gpurun_out/s4_tests.log
timeout 300 python tools/kbench.py unet > gpurun_out/s4_kbench_unet.txt 2>&1; cat gpurun_out/s4_kbench_unet.txt
bash tools/gpu_attn_akt.sh s4 > gpurun_out/s4_akt.txt 2>&1; cat gpurun_out/s4_akt.txt
timeout 900 python bench.py --workload c3 > gpurun_out/bench_c3_s4.json 2> gpurun_out/bench_c3_s4.err
python -c "import json; d=json.load(open('gpurun_out/bench_c3_s4.json')); print('c3', d['ms_per_step'], {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 9000 -c 3000 \
  --csv --log-file gpurun_out/launches_c3_s4.csv python bench.py --ncu --workload c3 \
  > gpurun_out/ncu_list_c3_s4.log 2>&1; echo "list rc=$?"
