r=16
timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20 > gpurun_out/r2ab.txt 2>&1
for d in 4 5; do echo -n "dbg$d "; DBL_FWD_DBG=$d timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done >> gpurun_out/r2ab.txt 2>&1
echo -n "dbg4 smem200 "; DBL_FWD_SMEM_KB=200 DBL_FWD_DBG=4 timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20 >> gpurun_out/r2ab.txt 2>&1
echo -n "dbg5 smem200 "; DBL_FWD_SMEM_KB=200 DBL_FWD_DBG=5 timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20 >> gpurun_out/r2ab.txt 2>&1
echo -n "smem200 "; DBL_FWD_SMEM_KB=200 timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20 >> gpurun_out/r2ab.txt 2>&1
cat gpurun_out/r2ab.txt
