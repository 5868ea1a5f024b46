# max-shared carveout so draft (72 KB) + target (154 KB) CTAs co-reside; DOUBLE bench
for kb in 154 180 200 227; do echo -n "smem$kb "; DBL_FWD_SMEM_KB=$kb timeout 300 python tools/fwd_probe.py qwen3-14b 17 288 20; done > gpurun_out/r2ad.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-side > gpurun_out/r2ad_bench.txt 2>&1
cat gpurun_out/r2ad.txt; tail -1 gpurun_out/r2ad_bench.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','ms_per_step','speedup_vs_ar','ar_tokens_per_s']}, d['e2e']['value'], d['roofline']['frac'], d['gamma_C']['value'], d['gamma_8']['value'])"
