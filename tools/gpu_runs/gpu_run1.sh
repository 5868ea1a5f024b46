set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_tp.py -x -q -s -m gpu 2>&1 | tail -40 > gpurun_out/g1_shapes.txt
timeout 1200 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_shapes.py 2>&1 | tail -15 > gpurun_out/g1_all.txt
cat gpurun_out/g1_shapes.txt gpurun_out/g1_all.txt
