# host probe + current forward timelines (planning the round-2 kernel work)
{ nproc; free -g; lscpu | grep -i "model name\|socket\|numa node(s)\|flags" | cut -c1-300; } > gpurun_out/r2c_host.txt 2>&1
python - >> gpurun_out/r2c_host.txt 2>&1 <<'PY'
import time, torch
print("torch threads", torch.get_num_threads())
for dt in (torch.bfloat16, torch.float32):
    W = torch.randn(17408, 5120, dtype=torch.float32).to(dt)
    x = torch.randn(2, 5120, dtype=torch.float32).to(dt)
    for _ in range(2): y = x @ W.T
    t = time.perf_counter(); n = 10
    for _ in range(n): y = x @ W.T
    dt_s = (time.perf_counter() - t) / n
    print(dt, f"{W.numel()*W.element_size()/dt_s/1e9:.1f} GB/s GEMV (2 rows)")
t = time.perf_counter(); A = torch.empty(1_000_000_000, dtype=torch.float32).normal_(0, 0.02); print("randn 1e9 fp32 s", time.perf_counter()-t)
PY
for r in 1 2 12 64; do DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b $r 288 > gpurun_out/r2c_tl_14b_$r.txt 2>&1; done
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-0.6b 11 288 > gpurun_out/r2c_tl_06b_11.txt 2>&1
for r in 1 2 12 64; do timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done > gpurun_out/r2c_probe.txt 2>&1
timeout 300 python tools/fwd_probe.py qwen3-0.6b 11 288 20 >> gpurun_out/r2c_probe.txt 2>&1
timeout 300 python tools/fwd_probe.py qwen3-0.6b 1 288 20 >> gpurun_out/r2c_probe.txt 2>&1
cat gpurun_out/r2c_host.txt gpurun_out/r2c_probe.txt
