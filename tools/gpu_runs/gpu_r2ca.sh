# A/B/C: attention with vectorized (permuted) K / V / q fragment loads (vec), and V held across token
# blocks of a group (grp), against the previous build (base)
mkdir -p gpurun_out
o=gpurun_out/r2ca_ab.txt; : > $o
# correctness first (a wrong kernel makes the timings moot)
for L in vec grp; do
  echo "== tests $L" >> $o
  DBL_LIB=$PWD/ab_libs/$L.so timeout 1500 python -m pytest tests/test_gpu_transformer.py tests/test_gpu_shapes.py tests/test_gpu_batch.py -x -q 2>&1 | tail -3 >> $o
done
for cfg in "qwen3-14b 2 288" "qwen3-14b 12 288" "qwen3-14b 24 288" "qwen3-14b 64 288" "qwen3-14b 12 1152" "qwen3-0.6b 11 288"; do
  set -- $cfg
  echo "== $cfg" >> $o
  for i in 1 2 3; do
    for L in base vec grp; do echo -n "$L " >> $o; DBL_LIB=$PWD/ab_libs/$L.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1; done
  done
done
cat $o
