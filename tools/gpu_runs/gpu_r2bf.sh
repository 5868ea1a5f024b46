R=400
for cfg in "1152 2" "1152 4" "1088 4" "1024 4" "1152 1"; do set -- $cfg; DBL_PREFILL_CHUNK=64 timeout 900 python tools/determinism_stress.py qwen3-0.6b $1 $2 $R; done 2>&1 | grep -v variant > gpurun_out/r2bf.txt
cat gpurun_out/r2bf.txt
