R=500
echo base > gpurun_out/r2bg.txt; DBL_PREFILL_CHUNK=64 timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 12 $R 2>&1 | grep -v variant >> gpurun_out/r2bg.txt
echo "per-thread fences" >> gpurun_out/r2bg.txt; DBL_FWD_DBG=11 DBL_PREFILL_CHUNK=64 timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 12 $R 2>&1 | grep -v variant >> gpurun_out/r2bg.txt
cat gpurun_out/r2bg.txt
