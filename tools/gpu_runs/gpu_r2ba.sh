R=200
timeout 900 python tools/determinism_stress.py qwen3-0.6b 1 200 $R > gpurun_out/r2ba.txt 2>&1
timeout 900 python tools/determinism_stress.py qwen3-0.6b 1 60 $R >> gpurun_out/r2ba.txt 2>&1
echo "chunk 64" >> gpurun_out/r2ba.txt; DBL_PREFILL_CHUNK=64 timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 12 $R >> gpurun_out/r2ba.txt 2>&1
echo "chunk 64, no early presum" >> gpurun_out/r2ba.txt; DBL_PREFILL_CHUNK=64 DBL_FWD_DBG=9 timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 12 $R >> gpurun_out/r2ba.txt 2>&1
cat gpurun_out/r2ba.txt
