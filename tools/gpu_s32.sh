# ncu --set full of the implicit 3x3 convs (stride 1: AM = 1, stride 2: AM = 2); summaries only
mkdir -p gpurun_out /tmp/ncu
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:\(int\)6, \(int\)3, \(int\)1>' -c 1 \
  -o /tmp/ncu/conv_s1 python tools/kbench.py conv > /tmp/ncu/s1.log 2>&1; echo "s1 rc=$?"
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k 'regex:\(int\)6, \(int\)3, \(int\)2>' -c 1 \
  -o /tmp/ncu/conv_s2 python tools/kbench.py unet > /tmp/ncu/s2.log 2>&1; echo "s2 rc=$?"
python tools/ncu_summary.py /tmp/ncu/conv_s1.ncu-rep /tmp/ncu/conv_s2.ncu-rep > gpurun_out/s32_conv_ncu.txt 2>&1
cat gpurun_out/s32_conv_ncu.txt | head -50
