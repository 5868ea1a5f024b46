for r in 1 2 12 64; do timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done > gpurun_out/r2g_probe.txt 2>&1
timeout 300 python tools/fwd_probe.py qwen3-14b 2 1152 20 >> gpurun_out/r2g_probe.txt 2>&1
timeout 300 python tools/fwd_probe.py qwen3-0.6b 11 288 20 >> gpurun_out/r2g_probe.txt 2>&1
timeout 300 python tools/fwd_probe.py qwen3-0.6b 1 288 20 >> gpurun_out/r2g_probe.txt 2>&1
cat gpurun_out/r2g_probe.txt
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 2 288 > gpurun_out/r2g_tl_14b_2.txt 2>&1
grep -A8 "layer 20 detail" gpurun_out/r2g_tl_14b_2.txt
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-0.6b 11 288 > gpurun_out/r2g_tl_06b_11.txt 2>&1
grep -A8 "layer 14 detail" gpurun_out/r2g_tl_06b_11.txt
