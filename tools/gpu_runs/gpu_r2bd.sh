R=400
for ctx in 65 129 300 600; do DBL_PREFILL_CHUNK=64 timeout 900 python tools/determinism_stress.py qwen3-0.6b $ctx 12 $R; done > gpurun_out/r2bd.txt 2>&1
cat gpurun_out/r2bd.txt | grep -v variant
