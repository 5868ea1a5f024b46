set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/r2a_gputest.txt
cat gpurun_out/r2a_gputest.txt
timeout 900 python bench.py > gpurun_out/r2a_bench.txt 2> gpurun_out/r2a_bench.err
tail -c 3000 gpurun_out/r2a_bench.txt; tail -20 gpurun_out/r2a_bench.err
