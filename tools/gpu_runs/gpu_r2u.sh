# graceful watchdog: tests + A/B (the waits now check for an abort every 128 polls)
timeout 900 python -m pytest tests/test_gpu_transformer.py tests/test_gpu_tp.py tests/test_gpu_table.py tests/test_gpu_multidev.py -x -q 2>&1 | tail -4 > gpurun_out/r2u.txt
for r in 2 12; do bash tools/ab_fwd.sh ab_libs/base.so ab_libs/new.so qwen3-14b $r 288; done >> gpurun_out/r2u.txt 2>&1
bash tools/ab_fwd.sh ab_libs/base.so ab_libs/new.so qwen3-0.6b 11 288 >> gpurun_out/r2u.txt 2>&1
cat gpurun_out/r2u.txt
