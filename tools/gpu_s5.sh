mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_unet.py -m gpu -q -p no:cacheprovider --timeout 400 -rfE > gpurun_out/s5_tests.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/s5_tests.log
timeout 300 python tools/kbench.py unet 2>&1 | grep groupnorm
CONV_IMPLICIT=1 timeout 300 python tools/kbench.py conv 2>&1
CONV_IMPLICIT=0 timeout 300 python tools/kbench.py conv 2>&1 | grep conv3x3
STADI_GEMM_MC=1 CONV_IMPLICIT=1 timeout 300 python tools/kbench.py conv 2>&1 | grep conv3x3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 \
  -o gpurun_out/s5_conv python tools/kbench.py conv > gpurun_out/s5_ncu_conv.log 2>&1; echo "ncu rc=$?"
for wl in c3 c4; do
  timeout 900 python bench.py --workload $wl > gpurun_out/bench_${wl}_s5.json 2> gpurun_out/bench_${wl}_s5.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${wl}_s5.json')); print('$wl', d['ms_per_step'], d['clocks'], {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"
done
