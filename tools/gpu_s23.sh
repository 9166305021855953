# DUAL_KV default 4096 (+ NARROW40 if adopted): full GPU suite + U-Net / C2 bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rfE > gpurun_out/s23_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/s23_tests.log
timeout 120 python tools/kbench.py small 2>&1
for v in 0 1 0 1; do echo "== DUAL40=$v"; STADI_ATTN_DUAL40=$v timeout 120 python tools/kbench.py attn 2>&1 | grep "hd=40"; done | tee gpurun_out/s23_dual40_ab.txt
for wl in c4 c3 c2; do
  timeout 900 python bench.py --workload $wl > gpurun_out/bench_${wl}_s23.json 2> gpurun_out/bench_${wl}_s23.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${wl}_s23.json')); print('$wl', d['ms_per_step'], d['clocks']['sm_mhz'], d['path_roofline']['frac'], {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"
done
