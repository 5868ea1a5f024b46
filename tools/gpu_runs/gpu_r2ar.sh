# A/B: the QKV epilogue in 32-column chunks too (16 < tp <= 64)
for r in 2 12 17 24 48 64; do bash tools/ab_fwd.sh ab_libs/base.so ab_libs/new.so qwen3-14b $r 288; done > gpurun_out/r2ar_ab.txt 2>&1
bash tools/ab_fwd.sh ab_libs/base.so ab_libs/new.so qwen3-0.6b 11 288 >> gpurun_out/r2ar_ab.txt 2>&1
DBL_LIB=$PWD/ab_libs/new.so timeout 1500 python -m pytest tests/test_gpu_transformer.py tests/test_gpu_shapes.py tests/test_gpu_batch.py tests/test_gpu_tp.py -x -q 2>&1 | tail -3 >> gpurun_out/r2ar_ab.txt
cat gpurun_out/r2ar_ab.txt
