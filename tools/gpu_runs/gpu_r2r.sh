timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_table.py tests/test_gpu_api.py -x -q -s 2>&1 | tail -8 > gpurun_out/r2r_index.txt
cat gpurun_out/r2r_index.txt
