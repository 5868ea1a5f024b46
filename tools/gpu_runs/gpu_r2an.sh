# which part of the second 16-column chunk costs at tp = 32 (16 tokens): 4 all, 5 none, 6 no partial writes,
# 7 no finisher chunk, 8 no early presum of chunk 2 (timing only)
timeout 300 python tools/fwd_probe.py qwen3-14b 16 288 20 > gpurun_out/r2an.txt 2>&1
for d in 4 5 6 7 8; do echo -n "dbg$d "; DBL_FWD_DBG=$d timeout 300 python tools/fwd_probe.py qwen3-14b 16 288 20; done >> gpurun_out/r2an.txt 2>&1
cat gpurun_out/r2an.txt
