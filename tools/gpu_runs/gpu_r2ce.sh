# A/B: attention softmax with the warp's four rows interleaved (smx), plus the combine phase taking two
# (token, q head) items per warp in lockstep (both) — same arithmetic, so logits must be bitwise equal
mkdir -p gpurun_out
o=gpurun_out/r2ce_ab.txt; : > $o
for L in base smx both; do DBL_LIB=$PWD/ab_libs/$L.so timeout 900 python tools/logits_hash.py > gpurun_out/r2ce_hash_$L.txt 2>&1; done
echo "bitwise smx vs base: $(cmp -s gpurun_out/r2ce_hash_base.txt gpurun_out/r2ce_hash_smx.txt && echo identical || echo DIFFERENT)" >> $o
echo "bitwise both vs base: $(cmp -s gpurun_out/r2ce_hash_base.txt gpurun_out/r2ce_hash_both.txt && echo identical || echo DIFFERENT)" >> $o
for cfg in "qwen3-14b 2 288" "qwen3-14b 12 288" "qwen3-14b 25 288" "qwen3-14b 64 288" "qwen3-14b 25 1152" "qwen3-0.6b 11 288"; do
  set -- $cfg
  echo "== $cfg" >> $o
  for i in 1 2 3; do
    for L in base smx both; do echo -n "$L " >> $o; DBL_LIB=$PWD/ab_libs/$L.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1; done
  done
done
cat $o
