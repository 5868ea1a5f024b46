rm -f /tmp/state.txt
DBL_DEBUG_STATE_FILE=/tmp/state.txt DBL_PREFILL_CHUNK=64 timeout 1500 python tools/determinism_stress.py qwen3-0.6b 1152 4 1500 > gpurun_out/r2bi.txt 2>&1
sort /tmp/state.txt | uniq -c | sort -rn | head -10 >> gpurun_out/r2bi.txt
cat gpurun_out/r2bi.txt
