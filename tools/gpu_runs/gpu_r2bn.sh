for d in 1 2 4; do DBL_DRAFT_GRID_DIV=$d timeout 900 python tools/draft_grid_probe.py; done > gpurun_out/r2bn.txt 2>&1
cat gpurun_out/r2bn.txt
