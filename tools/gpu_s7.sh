mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
bash tools/gpu_src_ab.sh tc_attn.cu tools/ab_tc_attn_head.cu attn "hd=72|hd=64|hd=40" 2>&1 | tee gpurun_out/s7_attn_ab.txt
bash tools/gpu_src_ab.sh tc_gemm.cu tools/ab_tc_gemm_head.cu gemm "." 2>&1 | tee gpurun_out/s7_gemm_ab.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 400 -rfE > gpurun_out/s7_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/s7_tests.log
for wl in c3 c2; do
  timeout 900 python bench.py --workload $wl > gpurun_out/bench_${wl}_s7.json 2> gpurun_out/bench_${wl}_s7.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${wl}_s7.json')); print('$wl', d['ms_per_step'], d['clocks'], {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"
done
