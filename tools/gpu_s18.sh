# ncu --set full of the C5 gated out-projection GEMM
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled \
  -k 'regex:\(int\)192, \(int\)2, \(int\)2' -s 10 -c 1 -o gpurun_out/s18_outproj python bench.py --steps 1 --warmup 3 --ncu \
  > gpurun_out/s18_ncu_outproj.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/s18_ncu_outproj.log; ls -la gpurun_out
