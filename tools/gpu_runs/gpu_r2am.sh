for k in 1 2 4; do echo -n "grid/$k "; DBL_FWD_GRID_DIV=$k timeout 300 python tools/fwd_probe.py qwen3-0.6b 11 288 20; done > gpurun_out/r2am.txt 2>&1
for k in 1 2 4; do echo -n "grid/$k "; DBL_FWD_GRID_DIV=$k DBL_FWD_SMEM_KB=200 timeout 300 python tools/fwd_probe.py qwen3-0.6b 11 288 20; done >> gpurun_out/r2am.txt 2>&1
for k in 1 2; do echo -n "grid/$k "; DBL_FWD_GRID_DIV=$k timeout 300 python tools/fwd_probe.py qwen3-14b 2 288 10; done >> gpurun_out/r2am.txt 2>&1
DBL_FWD_GRID_DIV=4 DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-0.6b 11 288 > gpurun_out/r2am_tl.txt 2>&1
cat gpurun_out/r2am.txt; grep -A9 "per phase kind" gpurun_out/r2am_tl.txt; grep -A7 "layer 14 detail" gpurun_out/r2am_tl.txt
