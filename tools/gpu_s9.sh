# implicit stride-2 / upsample convs + producer-zeroed edge halos: tests, bench lines, ncu of
# the U-Net HBM kernels (GN partials / apply, upsample) and the implicit convs
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_unet.py tests/test_gpu_fullres.py tests/test_gpu_ipc.py -m gpu -q -p no:cacheprovider --timeout 400 -rfE > gpurun_out/s9_tests.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/s9_tests.log
for wl in c3 c4; do
  timeout 900 python bench.py --workload $wl > gpurun_out/bench_${wl}_s9.json 2> gpurun_out/bench_${wl}_s9.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${wl}_s9.json')); print('$wl', d['ms_per_step'], d['clocks'], d.get('gpu_launches'), {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"
done
timeout 300 python tools/kbench.py unet 2>&1 | tee gpurun_out/s9_kbench_unet.txt
for k in gn_partials gn_apply upsample_pad im2col; do
  timeout 300 ncu --set full --clock-control none -k regex:$k -c 1 \
    -o gpurun_out/s9_$k python tools/kbench.py unet > gpurun_out/s9_ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
timeout 600 ncu --set full --clock-control none -k regex:tc_gemm -s 12 -c 2 \
  -o gpurun_out/s9_conv python tools/kbench.py unet > gpurun_out/s9_ncu_conv.log 2>&1; echo "ncu conv rc=$?"
