# A/B: tile-aligned stream-K split for phases with fewer tiles than CTAs (DBL_FWD_ALIGN=1: each tile
# gets exactly c = floor(active / tiles) contributors, every CTA's range inside one tile) vs the default
mkdir -p gpurun_out
o=gpurun_out/r2cd_ab.txt; : > $o
DBL_FWD_ALIGN=1 timeout 1500 python -m pytest tests/test_gpu_transformer.py tests/test_gpu_shapes.py -x -q 2>&1 | tail -2 >> $o
for cfg in "qwen3-14b 2 288" "qwen3-14b 12 288" "qwen3-14b 64 288" "qwen3-0.6b 11 288" "llama-3.3-70b 2 288"; do
  set -- $cfg
  echo "== $cfg" >> $o
  for i in 1 2 3; do
    for A in 0 1; do echo -n "align=$A " >> $o; DBL_FWD_ALIGN=$A timeout 300 python tools/fwd_probe.py $1 $2 $3 30 >> $o 2>&1; done
  done
done
DBL_FWD_ALIGN=1 DBL_FWD_TRACE=1 timeout 600 python tools/fwd_timeline.py qwen3-14b 2 288 > gpurun_out/r2cd_timeline_align_2rows.txt 2>&1
cat $o
