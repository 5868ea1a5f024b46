for r in 12 16; do timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; echo -n "tp32 "; DBL_FWD_DBG=4 timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done > gpurun_out/r2aa.txt 2>&1
echo -n "x16only "; DBL_FWD_DBG=1 timeout 300 python tools/fwd_probe.py qwen3-14b 17 288 20 >> gpurun_out/r2aa.txt 2>&1
timeout 300 python tools/fwd_probe.py qwen3-14b 17 288 20 >> gpurun_out/r2aa.txt 2>&1
cat gpurun_out/r2aa.txt
