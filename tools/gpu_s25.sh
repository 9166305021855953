# two-CTAs-per-SM attention at long K/V (C5 self-attention shape) A/B
mkdir -p gpurun_out
for v in 4096 16384 4096 16384; do echo "== DUAL_KV=$v"; STADI_ATTN_DUAL_KV=$v timeout 120 python tools/kbench.py attn 2>&1 | grep "hd=72\|hd=64"; STADI_ATTN_DUAL_KV=$v timeout 120 python -c "
import sys; sys.argv=['k']; sys.path.insert(0,'tools'); import kbench as K; K.attn(8192, 16384, 2, 16, 72); K.attn(2048, 16384, 2, 16, 72)"; done | tee gpurun_out/s25_dual_long_ab.txt
