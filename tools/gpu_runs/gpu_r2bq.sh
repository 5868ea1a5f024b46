# A/B: RoPE rows prefetched into L1 before the QKV head-norm reduction
for r in 2 12 24; do bash tools/ab_fwd.sh ab_libs/base.so ab_libs/new.so qwen3-14b $r 288; done > gpurun_out/r2bq.txt 2>&1
bash tools/ab_fwd.sh ab_libs/base.so ab_libs/new.so qwen3-0.6b 11 288 >> gpurun_out/r2bq.txt 2>&1
cat gpurun_out/r2bq.txt
