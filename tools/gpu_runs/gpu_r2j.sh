timeout 900 python -m pytest tests/test_gpu_transformer.py tests/test_gpu_shapes.py tests/test_gpu_batch.py tests/test_gpu_tp.py -x -q 2>&1 | tail -5
for r in 1 2 12 64; do timeout 300 python tools/fwd_probe.py qwen3-14b $r 288 20; done > gpurun_out/r2j_probe.txt 2>&1
timeout 300 python tools/fwd_probe.py qwen3-14b 2 1152 20 >> gpurun_out/r2j_probe.txt 2>&1
timeout 300 python tools/fwd_probe.py qwen3-0.6b 11 288 20 >> gpurun_out/r2j_probe.txt 2>&1
timeout 300 python tools/fwd_probe.py qwen3-0.6b 1 288 20 >> gpurun_out/r2j_probe.txt 2>&1
timeout 300 python tools/fwd_probe.py llama-3.1-8b 8 1100 20 >> gpurun_out/r2j_probe.txt 2>&1
cat gpurun_out/r2j_probe.txt
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 2 288 > gpurun_out/r2j_tl_14b_2.txt 2>&1
DBL_FWD_TRACE=1 timeout 300 python tools/fwd_timeline.py qwen3-14b 64 288 > gpurun_out/r2j_tl_14b_64.txt 2>&1
for f in gpurun_out/r2j_tl_14b_2.txt gpurun_out/r2j_tl_14b_64.txt; do grep -A8 "layer 20 detail" $f | head -8; tail -n 2 $f; done
