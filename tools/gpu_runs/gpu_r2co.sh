# A/B: the producer's bounded park while activations wait on a dependency, 250 ns (base) vs 40 ns
mkdir -p gpurun_out
o=gpurun_out/r2co_ab.txt; : > $o
for cfg in "qwen3-14b 1 288" "qwen3-14b 2 288" "qwen3-14b 12 288" "qwen3-14b 64 288" "qwen3-0.6b 11 288" "llama-3.3-70b 2 288"; do
  set -- $cfg
  echo "== $cfg" >> $o
  for i in 1 2 3; do for L in base h40; do echo -n "$L " >> $o; DBL_LIB=$PWD/ab_libs/$L.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1; done; done
done
cat $o
