mkdir -p gpurun_out
BUILD_VARIANTS="-DSTADI_ATTN_WARPMMA=0 base" bash tools/gpu_attn_build_ab.sh 2>&1 | tee gpurun_out/s6_ab.txt
python -m paper_2509_04719_b200.build > /dev/null 2>&1
timeout 300 python tools/kbench.py attn 2>&1 | tee -a gpurun_out/s6_ab.txt
timeout 300 python tools/kbench.py xattn 2>&1 | tee -a gpurun_out/s6_ab.txt
timeout 900 python bench.py > gpurun_out/bench_c5_s6.json 2> gpurun_out/bench_c5_s6.err
python -c "import json; d=json.load(open('gpurun_out/bench_c5_s6.json')); print('c5', d['ms_per_step'], d['clocks'], d['roofline']['achieved'], d['roofline']['frac'], {k:(v['launches'], round(v['ms']/d['steps'],1)) for k,v in d['kernels'].items()})"
