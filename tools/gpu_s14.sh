# C4 launch list (shares of the SDXL step; ncu serialises launches)
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 10000 -c 2500 --csv \
  --log-file gpurun_out/s14_c4_launches.csv python bench.py --steps 1 --warmup 3 --ncu --workload c4 > gpurun_out/s14_ncu_list.log 2>&1
echo "list rc=$?"; grep -c gpu__time gpurun_out/s14_c4_launches.csv
# ncu --set full of the C5 gated out-projection GEMM (HBM-bound fp32 residual RMW)
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:tc_gemm_kernel<192, 2, 2" -s 20 -c 1 \
  -o gpurun_out/s14_outproj python bench.py --steps 1 --warmup 3 --ncu > gpurun_out/s14_ncu_outproj.log 2>&1
echo "outproj rc=$?"
