# A/B: activation boxes (fewer producer copies) + early presum at tp > 16; then correctness tests
for r in 2 12 24 40 64; do bash tools/ab_fwd.sh ab_libs/base.so ab_libs/new.so qwen3-14b $r 288; done > gpurun_out/r2p_ab.txt 2>&1
bash tools/ab_fwd.sh ab_libs/base.so ab_libs/new.so qwen3-0.6b 11 288 >> gpurun_out/r2p_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_transformer.py tests/test_gpu_shapes.py tests/test_gpu_batch.py tests/test_gpu_tp.py -x -q 2>&1 | tail -3 >> gpurun_out/r2p_ab.txt
cat gpurun_out/r2p_ab.txt
