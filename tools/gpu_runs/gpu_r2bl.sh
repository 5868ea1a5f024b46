for i in 1 2; do for L in prefix fix; do echo -n "$L "; DBL_LIB=$PWD/ab_libs/$L.so timeout 600 python tools/gamma1_round_probe.py | tail -1; done; done > gpurun_out/r2bl.txt 2>&1
bash tools/ab_fwd.sh ab_libs/prefix.so ab_libs/fix.so qwen3-14b 2 288 >> gpurun_out/r2bl.txt 2>&1
cat gpurun_out/r2bl.txt
