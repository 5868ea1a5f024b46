for d in 1 4 8 2; do echo -n "draft grid /$d: "; DBL_DRAFT_GRID_DIV=$d timeout 600 python tools/gamma1_round_probe.py | tail -1; done > gpurun_out/r2bm.txt 2>&1
cat gpurun_out/r2bm.txt
