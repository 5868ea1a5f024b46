# A/B: the interleaved attention softmax (smx) and the same with the butterflies only for the warp's
# valid rows (smxg) vs base; logits must be bitwise equal
mkdir -p gpurun_out
o=gpurun_out/r2cf_ab.txt; : > $o
for L in base smxg; do DBL_LIB=$PWD/ab_libs/$L.so timeout 900 python tools/logits_hash.py > gpurun_out/r2cf_hash_$L.txt 2>&1; done
echo "bitwise smxg vs base: $(cmp -s gpurun_out/r2cf_hash_base.txt gpurun_out/r2cf_hash_smxg.txt && echo identical || echo DIFFERENT)" >> $o
for cfg in "qwen3-14b 2 288" "qwen3-14b 12 288" "qwen3-14b 25 288" "qwen3-14b 64 288"; do
  set -- $cfg
  echo "== $cfg" >> $o
  for i in 1 2 3 4; do
    for L in base smx smxg; do echo -n "$L " >> $o; DBL_LIB=$PWD/ab_libs/$L.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1; done
  done
done
cat $o
