for L in at_0362506 at_77f3a4d; do for r in 4 12; do DBL_LIB=$PWD/ab_libs/$L.so timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 $r 150; done; done > gpurun_out/r2ay.txt 2>&1
for r in 4 12; do timeout 900 python tools/determinism_stress.py qwen3-0.6b 1152 $r 150; done >> gpurun_out/r2ay.txt 2>&1
cat gpurun_out/r2ay.txt
