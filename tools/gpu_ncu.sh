# ncu evidence for one bench request: launch list (per-launch device time) and a
# --set full capture of the top kernels.  Usage: bash tools/gpu_ncu.sh <tag> [workload]
tag=${1:-r}; wl=${2:-c5}
mkdir -p gpurun_out
# launches of the profiling pass (skipped) then one whole request
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-1300} -c ${COUNT:-400} \
  --csv --log-file gpurun_out/launches_$tag.csv python bench.py --ncu --workload $wl \
  > gpurun_out/ncu_list_$tag.log 2>&1; echo "list rc=$?"
for k in ${KERNELS:-tc_attn tc_gemm}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s ${FSKIP:-40} -c 1 \
    -o gpurun_out/full_${k}_$tag python bench.py --ncu --workload $wl > gpurun_out/ncu_full_${k}_$tag.log 2>&1
  echo "full $k rc=$?"
done
ls -la gpurun_out
