timeout 600 python tools/determinism_stress.py qwen3-0.6b 1152 12 60 > gpurun_out/r2ax.txt 2>&1
DBL_FWD_SMEM_KB=113 timeout 600 python tools/determinism_stress.py qwen3-0.6b 1152 12 60 >> gpurun_out/r2ax.txt 2>&1
timeout 600 python tools/determinism_stress.py qwen3-0.6b 300 12 60 >> gpurun_out/r2ax.txt 2>&1
timeout 600 python tools/determinism_stress.py qwen3-0.6b 1152 4 60 >> gpurun_out/r2ax.txt 2>&1
cat gpurun_out/r2ax.txt
