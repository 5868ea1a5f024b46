R=200
echo "chunk 64" > gpurun_out/r2bb.txt; DBL_PREFILL_CHUNK=64 timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 12 $R >> gpurun_out/r2bb.txt 2>&1
timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 12 $R >> gpurun_out/r2bb.txt 2>&1
timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 4 $R >> gpurun_out/r2bb.txt 2>&1
for r in 2 12 64; do timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done >> gpurun_out/r2bb.txt 2>&1
timeout 300 python tools/fwd_probe.py qwen3-0.6b 11 288 20 >> gpurun_out/r2bb.txt 2>&1
cat gpurun_out/r2bb.txt
