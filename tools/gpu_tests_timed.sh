# GPU tests with per-test durations, U-Net first.  Usage: bash tools/gpu_tests_timed.sh <tag>
tag=${1:-r}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_unet.py tests/test_gpu_kernels.py tests/test_gpu_parity.py \
  -m gpu -q -p no:cacheprovider --timeout 300 --durations=25 -rfE > gpurun_out/tests_$tag.log 2>&1
echo "pytest rc=$?"; tail -90 gpurun_out/tests_$tag.log
