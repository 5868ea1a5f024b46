# A/B: skewed stream-K split (DBL_FWD_SKEW_X = X units: a tile's finisher takes X more 16 KiB units than
# its pure contributors, so their partials land before its own MMAs end) vs the uniform split (base)
mkdir -p gpurun_out
o=gpurun_out/r2ch_ab.txt; : > $o
DBL_FWD_SKEW_X=8 DBL_LIB=$PWD/ab_libs/skew.so timeout 1500 python -m pytest tests/test_gpu_transformer.py tests/test_gpu_shapes.py tests/test_gpu_batch.py -x -q 2>&1 | tail -2 >> $o
for cfg in "qwen3-14b 2 288" "qwen3-14b 12 288" "qwen3-14b 25 288" "qwen3-14b 64 288"; do
  set -- $cfg
  echo "== $cfg" >> $o
  for i in 1 2 3; do
    echo -n "base " >> $o; DBL_LIB=$PWD/ab_libs/base.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1
    for X in 0 4 8 12; do echo -n "x$X " >> $o; DBL_FWD_SKEW_X=$X DBL_LIB=$PWD/ab_libs/skew.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1; done
  done
done
echo "== llama-3.3-70b 2 288" >> $o
for i in 1 2; do
  echo -n "base " >> $o; DBL_LIB=$PWD/ab_libs/base.so timeout 300 python tools/fwd_probe.py llama-3.3-70b 2 288 30 >> $o 2>&1
  for X in 8 12; do echo -n "x$X " >> $o; DBL_FWD_SKEW_X=$X DBL_LIB=$PWD/ab_libs/skew.so timeout 300 python tools/fwd_probe.py llama-3.3-70b 2 288 30 >> $o 2>&1; done
done
DBL_FWD_SKEW_X=8 DBL_LIB=$PWD/ab_libs/skew.so DBL_FWD_TRACE=1 timeout 600 python tools/fwd_timeline.py qwen3-14b 2 288 > gpurun_out/r2ch_timeline_skew8_2rows.txt 2>&1
cat $o
