mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullres.py tests/test_gpu_parity.py tests/test_gpu_unet.py -m gpu -q -p no:cacheprovider > gpurun_out/s30_tests.log 2>&1
echo "pytest rc=$?"; tail -40 gpurun_out/s30_tests.log
