R=150
timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 12 $R > gpurun_out/r2az.txt 2>&1
for c in 128 64; do echo "chunk $c" >> gpurun_out/r2az.txt; DBL_PREFILL_CHUNK=$c timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 12 $R >> gpurun_out/r2az.txt 2>&1; done
echo "no early presum" >> gpurun_out/r2az.txt; DBL_FWD_DBG=9 timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 12 $R >> gpurun_out/r2az.txt 2>&1
cat gpurun_out/r2az.txt
