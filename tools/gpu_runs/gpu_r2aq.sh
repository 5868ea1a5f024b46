# A/B: smallest stream-K range per CTA (kFwdMinUnits 4 / 8 / 16): fewer split contributors in small phases
for L in base mu2 mu3; do for i in 1 2; do echo -n "$L "; DBL_LIB=$PWD/ab_libs/$L.so timeout 300 python tools/fwd_probe.py qwen3-0.6b 11 288 30; done; done > gpurun_out/r2aq.txt 2>&1
for L in base mu2 mu3; do echo -n "$L "; DBL_LIB=$PWD/ab_libs/$L.so timeout 300 python tools/fwd_probe.py llama-3.2-1b 11 1100 30; done >> gpurun_out/r2aq.txt 2>&1
for L in base mu2 mu3; do echo -n "$L "; DBL_LIB=$PWD/ab_libs/$L.so timeout 300 python tools/fwd_probe.py qwen3-14b 2 288 20; done >> gpurun_out/r2aq.txt 2>&1
cat gpurun_out/r2aq.txt
