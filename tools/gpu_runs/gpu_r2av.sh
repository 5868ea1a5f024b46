for mdl in qwen3-0.6b qwen3-32b; do timeout 600 python tools/determinism_probe.py $mdl 12; done > gpurun_out/r2av.txt 2>&1
echo "--- DBL_FWD_SMEM_KB=113" >> gpurun_out/r2av.txt
DBL_FWD_SMEM_KB=113 timeout 600 python tools/determinism_probe.py qwen3-0.6b 12 >> gpurun_out/r2av.txt 2>&1
cat gpurun_out/r2av.txt
