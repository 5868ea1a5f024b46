# final-state ncu --set full captures: the 2-row Qwen3-14B verify forward (the bench's per-forward shape)
# and a 25-row verify (the aligned workload's), plus the decode-path launch list of the bench command
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 2 -c 1 -o gpurun_out/r2cg_fwd14b_2rows \
    python tools/fwd_probe.py qwen3-14b 2 288 3 > gpurun_out/r2cg_ncu14b.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 2 -c 1 -o gpurun_out/r2cg_fwd14b_25rows \
    python tools/fwd_probe.py qwen3-14b 25 288 3 > gpurun_out/r2cg_ncu14b25.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/r2cg_launches.csv \
    timeout 900 python bench.py --steps 1 --warmup 1 --no-side --no-serving > gpurun_out/r2cg_launch_bench.txt 2>&1
ls -la gpurun_out/
