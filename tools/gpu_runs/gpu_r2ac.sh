# role-based shared-memory budgets (target 154 KB, draft 72 KB beside it): forwards + DOUBLE decodes
for r in 2 12 17 24 48 64; do timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done > gpurun_out/r2ac.txt 2>&1
for r in 1 11; do timeout 300 python tools/fwd_probe.py qwen3-0.6b $r 288 20; done >> gpurun_out/r2ac.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/r2ac.txt
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2ac_bench.txt 2>&1
cat gpurun_out/r2ac.txt; tail -c 4500 gpurun_out/r2ac_bench.txt
