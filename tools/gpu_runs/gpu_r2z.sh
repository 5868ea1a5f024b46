DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 24 288 > gpurun_out/r2z_tl_14b_24.txt 2>&1
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 16 288 > gpurun_out/r2z_tl_14b_16.txt 2>&1
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 17 288 > gpurun_out/r2z_tl_14b_17.txt 2>&1
for f in gpurun_out/r2z_tl_14b_16.txt gpurun_out/r2z_tl_14b_17.txt gpurun_out/r2z_tl_14b_24.txt; do head -1 $f; grep -A10 "per phase kind" $f; grep -A8 "layer 20 detail" $f; done
