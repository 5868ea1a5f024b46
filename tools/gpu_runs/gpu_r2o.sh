# row sweep of the 14B verify forward + timeline at 24 rows
for r in 1 8 12 16 17 24 32 40 48 64; do timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done > gpurun_out/r2o_rows.txt 2>&1
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 24 288 > gpurun_out/r2o_tl_14b_24.txt 2>&1
cat gpurun_out/r2o_rows.txt
