# forward timelines: draft (0.6B, 11 rows) and target (14B, 2 and 64 rows)
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-0.6b 11 288 > gpurun_out/r2l_tl_06b_11.txt 2>&1
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 2 288 > gpurun_out/r2l_tl_14b_2.txt 2>&1
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 64 288 > gpurun_out/r2l_tl_14b_64.txt 2>&1
cat gpurun_out/r2l_tl_06b_11.txt
