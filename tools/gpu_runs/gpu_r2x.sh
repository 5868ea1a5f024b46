for r in 12 24 48; do echo -n "x16only "; DBL_FWD_DBG=1 timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done > gpurun_out/r2x.txt 2>&1
for r in 12 24 48; do timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done >> gpurun_out/r2x.txt 2>&1
cat gpurun_out/r2x.txt
