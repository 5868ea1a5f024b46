timeout 900 python -m pytest tests/test_gpu_multidev.py -x -q 2>&1 | tail -15 > gpurun_out/r2t.txt
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 >> gpurun_out/r2t.txt
cat gpurun_out/r2t.txt
