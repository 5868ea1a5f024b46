# exact sampling at V = 151,936 against the reference loop; the sampled suite with defaults; C++ mirror
mkdir -p gpurun_out
o=gpurun_out/r2cj.txt
timeout 1800 python -m pytest tests/test_gpu_sampled.py -q --durations=6 2>&1 | tail -12 > $o
timeout 300 ./build/test_cpp_api >> $o 2>&1; echo "test_cpp_api rc=$?" >> $o
cat $o
