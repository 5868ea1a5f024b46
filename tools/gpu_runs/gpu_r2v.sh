# r2v: launch list of the bench command, one ncu --set full capture of the 2-row 14B fwd_kernel and of the
# 11-row 0.6B draft forward, compute-sanitizer memcheck / racecheck / synccheck on the tiny transformer path
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/r2v_launches.csv \
    timeout 900 python bench.py --steps 1 --warmup 1 --no-side --no-serving > gpurun_out/r2v_launch_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 2 -c 1 -o gpurun_out/r2v_fwd14b \
    python tools/fwd_probe.py qwen3-14b 2 288 3 > gpurun_out/r2v_ncu14b.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -s 2 -c 1 -o gpurun_out/r2v_fwd06b \
    python tools/fwd_probe.py qwen3-0.6b 11 288 3 > gpurun_out/r2v_ncu06b.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py > gpurun_out/r2v_san_$tool.txt 2>&1
  echo "$tool exit $?" >> gpurun_out/r2v_san_summary.txt
  tail -3 gpurun_out/r2v_san_$tool.txt >> gpurun_out/r2v_san_summary.txt
done
cat gpurun_out/r2v_san_summary.txt
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_fwd_probe.py > gpurun_out/r2v_sanfwd_$tool.txt 2>&1
  echo "fwd $tool exit $?" >> gpurun_out/r2v_san_summary.txt
  tail -3 gpurun_out/r2v_sanfwd_$tool.txt >> gpurun_out/r2v_san_summary.txt
done
cat gpurun_out/r2v_san_summary.txt
