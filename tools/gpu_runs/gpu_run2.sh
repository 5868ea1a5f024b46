timeout 900 python -m pytest tests/test_gpu_transformer.py -x -q -k "above_256 or logits_match" 2>&1 | tail -15 > gpurun_out/g2_split.txt
timeout 1500 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_tp.py -q -s -m gpu 2>&1 | grep -v "^$" | tail -60 > gpurun_out/g2_shapes.txt
cat gpurun_out/g2_split.txt gpurun_out/g2_shapes.txt
