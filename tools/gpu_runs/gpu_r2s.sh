timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_table.py tests/test_gpu_api.py tests/test_gpu_batch.py -x -q -s 2>&1 | tail -5 > gpurun_out/r2s.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-side > gpurun_out/r2s_bench.txt 2>&1
cat gpurun_out/r2s.txt; tail -c 2500 gpurun_out/r2s_bench.txt
