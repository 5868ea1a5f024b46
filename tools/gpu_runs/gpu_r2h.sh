DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 2 288 > gpurun_out/r2h_tl_14b_2.txt 2>&1
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-0.6b 11 288 > gpurun_out/r2h_tl_06b_11.txt 2>&1
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 64 288 > gpurun_out/r2h_tl_14b_64.txt 2>&1
tail -4 gpurun_out/r2h_tl_14b_2.txt gpurun_out/r2h_tl_06b_11.txt gpurun_out/r2h_tl_14b_64.txt
