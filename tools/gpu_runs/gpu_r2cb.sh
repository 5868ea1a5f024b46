# per-phase timelines of the verify forward at 2 and 12 rows (current state), and the draft at 11
mkdir -p gpurun_out
DBL_FWD_TRACE=1 timeout 600 python tools/fwd_timeline.py qwen3-14b 2 288 > gpurun_out/r2cb_timeline_2rows.txt 2>&1
DBL_FWD_TRACE=1 timeout 600 python tools/fwd_timeline.py qwen3-14b 12 288 > gpurun_out/r2cb_timeline_12rows.txt 2>&1
DBL_FWD_TRACE=1 timeout 600 python tools/fwd_timeline.py qwen3-0.6b 11 288 > gpurun_out/r2cb_timeline_draft11.txt 2>&1
head -3 gpurun_out/r2cb_timeline_2rows.txt
