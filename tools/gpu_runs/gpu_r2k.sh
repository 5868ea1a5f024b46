# round-2 state check after re-entry: full -m gpu suite, smoke, forward probes, short bench
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2k_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.txt 2>&1
for r in 1 2 12 64; do timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done > gpurun_out/r2k_probe.txt 2>&1
for r in 1 11; do timeout 300 python tools/fwd_probe.py qwen3-0.6b $r 288 20; done >> gpurun_out/r2k_probe.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2k_bench.txt 2>&1
cat gpurun_out/r2k_gputest.txt gpurun_out/r2k_smoke.txt gpurun_out/r2k_probe.txt; tail -c 3000 gpurun_out/r2k_bench.txt
