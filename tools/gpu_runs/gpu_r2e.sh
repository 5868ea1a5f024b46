DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 2 288 > gpurun_out/r2e_tl_14b_2.txt 2>&1
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 64 288 > gpurun_out/r2e_tl_14b_64.txt 2>&1
head -60 gpurun_out/r2e_tl_14b_2.txt
grep -A3 "layer 20 detail" gpurun_out/r2e_tl_14b_64.txt; grep "attention" gpurun_out/r2e_tl_14b_64.txt
