timeout 900 python -m pytest tests/test_gpu_transformer.py -x -q -k "above_256" 2>&1 | tail -15 > gpurun_out/g3_split.txt
cat gpurun_out/g3_split.txt
