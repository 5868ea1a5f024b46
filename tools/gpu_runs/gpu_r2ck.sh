# closing validation: -m gpu suite, smoke, default bench, reference arm
mkdir -p gpurun_out
o=gpurun_out/r2ck.txt
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $o
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $o 2>&1
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2ck_bench.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2ck_ref.txt 2>&1
cat $o; tail -1 gpurun_out/r2ck_bench.txt | cut -c1-300; tail -1 gpurun_out/r2ck_ref.txt | cut -c1-200
