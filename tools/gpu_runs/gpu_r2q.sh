# A/B: box 16 for all T <= 16 vs 4/8/16; and a deeper ring (DBL_FWD_SMEM_KB) at 2 / 24 / 64 rows
for r in 2 12; do bash tools/ab_fwd.sh ab_libs/new.so ab_libs/b16.so qwen3-14b $r 288; done > gpurun_out/r2q_ab.txt 2>&1
for kb in 113 160 200; do for r in 2 24 64; do echo -n "smem $kb "; DBL_FWD_SMEM_KB=$kb timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 30; done; done >> gpurun_out/r2q_ab.txt 2>&1
cat gpurun_out/r2q_ab.txt
