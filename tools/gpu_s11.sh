# GN apply (fixed vector per thread, tanh SiLU) + GEMM cost-model L2 bandwidth A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_unet.py -m gpu -q -p no:cacheprovider --timeout 300 -rfE > gpurun_out/s11_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/s11_tests.log
timeout 300 python tools/kbench.py unet 2>&1 | grep groupnorm
for l2 in 6300 9000 12600 20000; do echo "== L2=$l2"; STADI_GEMM_L2=$l2 timeout 300 python tools/kbench.py unet 2>&1 | grep -E "^gemm|mode=0|^conv3x3 [0-9]|implicit=1"; done | tee gpurun_out/s11_l2_ab.txt
for l2 in 6300 12600; do STADI_GEMM_L2=$l2 timeout 900 python bench.py --workload c4 --no-method --no-occ-sweep > gpurun_out/bench_c4_s11_$l2.json 2> gpurun_out/bench_c4_s11_$l2.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_s11_$l2.json')); print('c4 L2=$l2', d['ms_per_step'], d['clocks'], {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"; done
for l2 in 6300 12600; do STADI_GEMM_L2=$l2 timeout 900 python bench.py --workload c3 --no-method --no-occ-sweep > gpurun_out/bench_c3_s11_$l2.json 2> gpurun_out/bench_c3_s11_$l2.err
python -c "import json; d=json.load(open('gpurun_out/bench_c3_s11_$l2.json')); print('c3 L2=$l2', d['ms_per_step'], d['clocks'], {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"; done
