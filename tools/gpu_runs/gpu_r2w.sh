# r2w: where the 17+-row forward loses (activation traffic? attention?), decode-path launch list
for r in 2 12 24 48; do timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done > gpurun_out/r2w_rows.txt 2>&1
for r in 2 12 24 48; do echo -n "noX "; DBL_FWD_DBG=1 timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done >> gpurun_out/r2w_rows.txt 2>&1
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 12 288 > gpurun_out/r2w_tl_14b_12.txt 2>&1
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 24 288 > gpurun_out/r2w_tl_14b_24.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 900 -c 3000 --csv --log-file gpurun_out/r2w_launches.csv \
    timeout 900 python bench.py --steps 1 --warmup 1 --no-side --no-serving > gpurun_out/r2w_launch_bench.txt 2>&1
cat gpurun_out/r2w_rows.txt
for f in gpurun_out/r2w_tl_14b_12.txt gpurun_out/r2w_tl_14b_24.txt; do grep -A10 "per phase kind" $f; done
