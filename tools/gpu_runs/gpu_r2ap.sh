DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 64 288 > gpurun_out/r2ap_tl_64.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 2 -c 1 -o gpurun_out/r2ap_fwd14b_r12 python tools/fwd_probe.py qwen3-14b 12 288 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 2 -c 1 -o gpurun_out/r2ap_fwd14b_r64 python tools/fwd_probe.py qwen3-14b 64 288 3 > /dev/null 2>&1
grep -A10 "per phase kind" gpurun_out/r2ap_tl_64.txt; grep -A7 "layer 20 detail" gpurun_out/r2ap_tl_64.txt; tail -3 gpurun_out/r2ap_tl_64.txt
