R=400
echo "chunk 64 base" > gpurun_out/r2bc.txt; DBL_PREFILL_CHUNK=64 timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 12 $R >> gpurun_out/r2bc.txt 2>&1
echo "chunk 64 no L2 warm" >> gpurun_out/r2bc.txt; DBL_PREFILL_CHUNK=64 DBL_FWD_DBG=10 timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 12 $R >> gpurun_out/r2bc.txt 2>&1
cat gpurun_out/r2bc.txt
