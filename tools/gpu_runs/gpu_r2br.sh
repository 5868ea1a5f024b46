timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r2br.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r2br.txt 2>&1
timeout 1200 python bench.py --steps 3 --warmup 3 --log-out bench_data/qwen3-0.6b_qwen3-14b.json > gpurun_out/r2br_bench.txt 2>&1
mkdir -p gpurun_out/bench_data; cp bench_data/qwen3-0.6b_qwen3-14b.json gpurun_out/bench_data/
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2br_ref.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 900 -c 3000 --csv --log-file gpurun_out/r2br_launches.csv \
    timeout 900 python bench.py --steps 1 --warmup 1 --no-side --no-serving > /dev/null 2>&1
cat gpurun_out/r2br.txt; tail -1 gpurun_out/r2br_bench.txt | cut -c1-300; tail -1 gpurun_out/r2br_ref.txt | cut -c1-200
