# A/B of the attention kernel's run-time switches (tc_attn.cu attn_flags) on the C5 shape
for v in "TOK=1" "TOK=0" "TOK=0 ORDER=1" "TOK=0 DEFER=0" "TOK=0 TOK4=1" "TOK=1 ORDER=1"; do
  envs=""; for kv in $v; do envs="$envs STADI_ATTN_$kv"; done
  for i in 1 2; do r=$(env $envs timeout 120 python tools/kbench.py attn 2>&1 | grep "hd=72"); echo "$v: $r"; done
done
