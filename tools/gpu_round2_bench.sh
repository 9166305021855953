# Round-2 measurement: the default bench line (as the driver runs it), the ncu launch
# list of the same command (per-launch times, cold and serialised: shares only), and
# one ncu --set full capture of the attention kernel.
set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -3 gpurun_out/r2_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 22000 -c 6000 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 3 --ncu > gpurun_out/r2_ncu_list.log 2>&1
tail -3 gpurun_out/r2_ncu_list.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -s 200 -c 1 -o gpurun_out/r2_attn python bench.py --steps 1 --warmup 3 --ncu > gpurun_out/r2_ncu_full.log 2>&1
tail -3 gpurun_out/r2_ncu_full.log
ls -la gpurun_out
