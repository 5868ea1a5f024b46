# what paces a CTA's weight stream?  timing probes (results invalid): DBL_FWD_DBG=13 issues 1 of the 4
# MMAs per 16 KiB stage, 14 none (the stage is freed by the commit alone), plus a deeper ring (200 KB)
mkdir -p gpurun_out
o=gpurun_out/r2cl_probe.txt; : > $o
for cfg in "qwen3-14b 2 288" "qwen3-14b 64 288"; do
  set -- $cfg
  echo "== $cfg" >> $o
  for i in 1 2; do
    echo -n "4mma " >> $o; DBL_LIB=$PWD/ab_libs/probe.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1
    echo -n "1mma " >> $o; DBL_FWD_DBG=13 DBL_LIB=$PWD/ab_libs/probe.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1
    echo -n "0mma " >> $o; DBL_FWD_DBG=14 DBL_LIB=$PWD/ab_libs/probe.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1
    echo -n "0mma+200KB " >> $o; DBL_FWD_SMEM_KB=200 DBL_FWD_DBG=14 DBL_LIB=$PWD/ab_libs/probe.so timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1
  done
done
DBL_FWD_DBG=14 DBL_LIB=$PWD/ab_libs/probe.so DBL_FWD_TRACE=1 timeout 600 python tools/fwd_timeline.py qwen3-14b 2 288 > gpurun_out/r2cl_timeline_0mma.txt 2>&1
cat $o
