python tools/kbench.py 2>&1 | grep gemm
for p in 0 2 3 4; do echo "POLY=$p"; STADI_ATTN_POLY=$p python tools/kbench.py 2>&1 | grep attn; done
