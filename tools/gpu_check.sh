# One gpurun call: GPU test suite, smoke, a bench line.  Usage: bash tools/gpu_check.sh [tag]
tag=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 300 \
  > gpurun_out/tests_$tag.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/tests_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
echo "smoke rc=$?"; tail -3 gpurun_out/smoke_$tag.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench rc=$?"; tail -3 gpurun_out/bench_$tag.err; head -c 1500 gpurun_out/bench_$tag.json
