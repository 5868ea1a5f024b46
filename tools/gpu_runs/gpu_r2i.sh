timeout 900 ncu --section SourceCounters --section WarpStateStats --section SchedulerStats -k regex:fwd_kernel -s 4 -c 1 --import-source on -f -o gpurun_out/r2i_ncu python tools/fwd_probe.py qwen3-14b 2 288 1 > gpurun_out/r2i_ncu.log 2>&1
tail -5 gpurun_out/r2i_ncu.log
ls -la gpurun_out/
