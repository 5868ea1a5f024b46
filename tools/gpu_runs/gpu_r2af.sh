# ring-depth sensitivity per role: 70B-shaped target (1 row) and 0.6B draft (11 rows)
for kb in 113 136 154 200; do echo -n "smem$kb "; DBL_FWD_SMEM_KB=$kb timeout 600 python tools/fwd_probe.py llama-3.3-70b 1 1152 10; done > gpurun_out/r2af.txt 2>&1
for kb in 72 90 113; do echo -n "smem$kb "; DBL_FWD_SMEM_KB=$kb timeout 300 python tools/fwd_probe.py qwen3-0.6b 11 288 20; done >> gpurun_out/r2af.txt 2>&1
for kb in 113 136 154; do echo -n "smem$kb "; DBL_FWD_SMEM_KB=$kb timeout 300 python tools/fwd_probe.py qwen3-14b 2 288 20; done >> gpurun_out/r2af.txt 2>&1
cat gpurun_out/r2af.txt
