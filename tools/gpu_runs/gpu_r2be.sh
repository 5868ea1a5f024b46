export DBL_FWD_WATCHDOG_MS=600000
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 python tools/determinism_stress.py qwen3-0.6b 1152 12 3 > gpurun_out/r2be_memcheck.txt 2>&1
tail -30 gpurun_out/r2be_memcheck.txt
