# final-state validation (NVTX build): -m gpu suite, smoke, the C++ mirror test, default bench, reference arm
mkdir -p gpurun_out
o=gpurun_out/r2cc.txt
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $o
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $o 2>&1
timeout 300 ./build/test_cpp_api >> $o 2>&1; echo "test_cpp_api rc=$?" >> $o
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2cc_bench.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2cc_ref.txt 2>&1
cat $o; tail -1 gpurun_out/r2cc_bench.txt | cut -c1-400; tail -1 gpurun_out/r2cc_ref.txt | cut -c1-200
