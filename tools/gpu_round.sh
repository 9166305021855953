# Tests + smoke + bench + ncu evidence in one gpurun call.  Usage: bash tools/gpu_round.sh <tag>
tag=${1:-r}
mkdir -p gpurun_out
bash tools/gpu_tests_timed.sh $tag
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$tag.log
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench rc=$?"; tail -3 gpurun_out/bench_$tag.err
bash tools/gpu_ncu.sh $tag c5
