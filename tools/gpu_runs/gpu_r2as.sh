timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r2as.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r2as.txt 2>&1
timeout 1200 python bench.py > gpurun_out/r2as_bench.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2as_ref.txt 2>&1
cat gpurun_out/r2as.txt; tail -1 gpurun_out/r2as_bench.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','ms_per_step','speedup_vs_ar','ar_tokens_per_s','steps','warmup']}, d['e2e']['value'], d['roofline']['frac'], d['clocks']); s=d['side_workloads']; print({k:(v.get('value'), v.get('speedup_vs_ar'), v.get('roofline',{}).get('frac')) for k,v in s.items()})"; tail -1 gpurun_out/r2as_ref.txt | cut -c1-400
