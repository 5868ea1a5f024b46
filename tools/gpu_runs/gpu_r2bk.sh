for i in 1 2; do timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3; done > gpurun_out/r2bk.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r2bk.txt 2>&1
timeout 1200 python bench.py > gpurun_out/r2bk_bench.txt 2>&1
cat gpurun_out/r2bk.txt; tail -1 gpurun_out/r2bk_bench.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','ms_per_step','speedup_vs_ar','ar_tokens_per_s']}, d['e2e']['value'], d['roofline']['frac'], d['clocks']); s=d['side_workloads']; print({k:(v.get('value'), v.get('speedup_vs_ar'), v.get('roofline',{}).get('frac')) for k,v in s.items()})"
