for L in at_0362506 at_77f3a4d at_98a5d1e at_bc42983; do DBL_LIB=$PWD/ab_libs/$L.so timeout 600 python tools/determinism_stress.py qwen3-0.6b 1152 12 40; done > gpurun_out/r2aw.txt 2>&1
DBL_FWD_SMEM_KB=113 timeout 600 python tools/determinism_stress.py qwen3-0.6b 1152 12 40 >> gpurun_out/r2aw.txt 2>&1
timeout 600 python tools/determinism_stress.py qwen3-0.6b 1152 12 40 >> gpurun_out/r2aw.txt 2>&1
timeout 600 python tools/determinism_stress.py qwen3-0.6b 1152 1 40 >> gpurun_out/r2aw.txt 2>&1
cat gpurun_out/r2aw.txt
