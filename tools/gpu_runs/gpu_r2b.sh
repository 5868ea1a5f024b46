set -x
timeout 600 python -m pytest tests/test_gpu_api.py tests/test_gpu_cpp_api.py -x -q 2>&1 | tail -30 > gpurun_out/r2b_api.txt
cat gpurun_out/r2b_api.txt
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/r2b_all.txt
cat gpurun_out/r2b_all.txt
