set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 22000 -c 6000 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 1 --warmup 3 --no-uniform --no-e2e --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
tail -3 gpurun_out/ncu_list.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -s 200 -c 1 -o gpurun_out/attn1 python bench.py --steps 1 --warmup 3 --no-uniform --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
