# functional check of the N = 2 bench path (torchrun, IPC transport) on a 1-GPU box (both
# ranks share the device: NOT a performance number), and attention exp-offload A/B
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --workload c2 --occupancy zero \
  --no-occ-sweep --no-method > gpurun_out/s12_n2_c2.json 2> gpurun_out/s12_n2_c2.err
echo "n2 rc=$?"; tail -c 600 gpurun_out/s12_n2_c2.json; tail -3 gpurun_out/s12_n2_c2.err
for v in "STADI_ATTN_POLY=0" "STADI_ATTN_POLY=1" "STADI_ATTN_POLY=2" "STADI_ATTN_POLY=1,STADI_ATTN_TOK4=0" "STADI_ATTN_POLY=2,STADI_ATTN_TOK4=0" "STADI_ATTN_TOK4=0"; do
  echo "== $v"; env ${v//,/ } timeout 120 python tools/kbench.py attn 2>&1 | grep "hd=72"
done | tee gpurun_out/s12_poly_ab.txt
# (compute-sanitizer is closed on the GPU pool: 'runs under it have left GPUs needing a
# reset' -- the kernels rely on bounds-checked parity tests instead)
