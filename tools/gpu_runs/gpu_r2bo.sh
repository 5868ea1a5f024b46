timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r2bo.txt
timeout 1200 python bench.py > gpurun_out/r2bo_bench.txt 2>&1
timeout 900 python tools/round_timeline.py gpurun_out/r2bo_round_timeline.jsonl > gpurun_out/r2bo_round_timeline.txt 2>&1
cat gpurun_out/r2bo.txt; tail -1 gpurun_out/r2bo_bench.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','ms_per_step','speedup_vs_ar','ar_tokens_per_s']}, d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['gamma_C'], d['gamma_8']); s=d['side_workloads']; print({k:(v.get('value'), v.get('speedup_vs_ar'), v.get('roofline',{}).get('frac')) for k,v in s.items()})"; head -6 gpurun_out/r2bo_round_timeline.txt
