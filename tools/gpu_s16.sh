# split-K/V attention for small grids: parity, microbench A/B, bench lines A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_unet.py tests/test_gpu_fullres.py -m gpu -q -p no:cacheprovider --timeout 400 -rfE > gpurun_out/s16_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/s16_tests.log
for v in 0 1 0 1; do echo "== SPLITKV=$v"; STADI_ATTN_SPLITKV=$v timeout 120 python tools/kbench.py small 2>&1; done | tee gpurun_out/s16_splitkv_ab.txt
timeout 120 python tools/kbench.py attn 2>&1 | grep hd=72 | tee -a gpurun_out/s16_splitkv_ab.txt
Q="--no-method --no-occ-sweep --no-cpu-baseline --no-uniform --no-e2e"
for wl in c2 c3 c4; do for v in 0 1; do
  STADI_ATTN_SPLITKV=$v timeout 900 python bench.py --workload $wl $Q > gpurun_out/bench_${wl}_s16_$v.json 2> gpurun_out/bench_${wl}_s16_$v.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${wl}_s16_$v.json')); print('$wl SPLITKV=$v', d['ms_per_step'], d['clocks']['sm_mhz'], {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"
done; done
