R=1500
for cfg in "1152 4" "1152 12" "1152 1"; do set -- $cfg; DBL_PREFILL_CHUNK=64 timeout 1200 python tools/determinism_stress.py qwen3-0.6b $1 $2 $R; done 2>&1 | grep -v variant > gpurun_out/r2bj.txt
rm -f /tmp/state.txt; DBL_DEBUG_STATE_FILE=/tmp/state.txt DBL_PREFILL_CHUNK=64 timeout 1500 python tools/determinism_stress.py qwen3-0.6b 1152 4 1500 2>&1 | grep -v variant >> gpurun_out/r2bj.txt
sort /tmp/state.txt | uniq -c | sort -rn | head -5 | cut -c1-120 >> gpurun_out/r2bj.txt
cat gpurun_out/r2bj.txt
