# exact-HEAD GPU suite
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -rfE > gpurun_out/s29_tests.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/s29_tests.log
