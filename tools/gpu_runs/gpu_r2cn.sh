# A/B: a stage's four MMAs issued from one asm block (descriptor offsets computed up front) vs base
mkdir -p gpurun_out
o=gpurun_out/r2cn_ab.txt; : > $o
for L in base k64; do DBL_LIB=$PWD/ab_libs/$L.so timeout 900 python tools/logits_hash.py > gpurun_out/r2cn_hash_$L.txt 2>&1; done
echo "bitwise k64 vs base: $(cmp -s gpurun_out/r2cn_hash_base.txt gpurun_out/r2cn_hash_k64.txt && echo identical || echo DIFFERENT)" >> $o
for cfg in "qwen3-14b 1 288" "qwen3-14b 2 288" "qwen3-14b 12 288" "qwen3-14b 25 288" "qwen3-14b 64 288" "qwen3-0.6b 11 288"; do
  set -- $cfg
  echo "== $cfg" >> $o
  for i in 1 2 3; do for L in base k64; do echo -n "$L " >> $o; DBL_LIB=$PWD/ab_libs/$L.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1; done; done
done
cat $o
