# experiment: is the per-CTA weight stream paced by the dependent MMA chain?  DBL_FWD_DBG=12 alternates
# each k-block's 4 MMAs between two TMEM accumulators (tp = 16 only), halving the accumulate chain
mkdir -p gpurun_out
o=gpurun_out/r2ci_ab.txt; : > $o
for cfg in "qwen3-14b 1 288" "qwen3-14b 2 288" "qwen3-14b 12 288" "qwen3-0.6b 11 288" "llama-3.3-70b 2 288"; do
  set -- $cfg
  echo "== $cfg" >> $o
  for i in 1 2 3; do
    echo -n "base " >> $o; DBL_LIB=$PWD/ab_libs/base.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1
    echo -n "single " >> $o; DBL_LIB=$PWD/ab_libs/dual.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1
    echo -n "dual " >> $o; DBL_FWD_DBG=12 DBL_LIB=$PWD/ab_libs/dual.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1
    echo -n "dual+skew8 " >> $o; DBL_FWD_SKEW_X=8 DBL_FWD_DBG=12 DBL_LIB=$PWD/ab_libs/dual.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1
  done
done
DBL_FWD_DBG=12 DBL_LIB=$PWD/ab_libs/dual.so DBL_FWD_TRACE=1 timeout 600 python tools/fwd_timeline.py qwen3-14b 2 288 > gpurun_out/r2ci_timeline_dual_2rows.txt 2>&1
DBL_FWD_DBG=12 DBL_LIB=$PWD/ab_libs/dual.so timeout 900 python tools/logits_hash.py > gpurun_out/r2ci_hash_dual.txt 2>&1
head -4 gpurun_out/r2ci_hash_dual.txt >> $o
cat $o
