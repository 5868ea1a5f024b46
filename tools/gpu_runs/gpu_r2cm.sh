# ring depth with the current build: 136 KB (default target budget) vs 160 / 200 / 227 KB
mkdir -p gpurun_out
o=gpurun_out/r2cm_ring.txt; : > $o
for r in 2 12; do for i in 1 2; do for kb in 0 160 200 227; do
  if [ $kb = 0 ]; then echo -n "136 " >> $o; DBL_LIB=$PWD/ab_libs/base.so timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 30 >> $o 2>&1;
  else echo -n "$kb " >> $o; DBL_FWD_SMEM_KB=$kb DBL_LIB=$PWD/ab_libs/base.so timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 30 >> $o 2>&1; fi
done; done; done
cat $o
