timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r2ag.txt
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2ag_bench.txt 2>&1
cat gpurun_out/r2ag.txt; tail -1 gpurun_out/r2ag_bench.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','ms_per_step','speedup_vs_ar','ar_tokens_per_s']}, d['e2e']['value'], d['roofline']['frac'], d['roofline']['draft_forward'], d['gamma_C']['value'], d['gamma_8']['value']); s=d['side_workloads']; print({k:(v.get('value'), v.get('speedup_vs_ar'), v.get('roofline',{}).get('frac')) for k,v in s.items()}); print(s['aligned-qwen3-14b'].get('gammas'))"
