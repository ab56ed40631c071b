# pair kernel: parity + timing vs the row-group kernel
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_r2.py -q -m gpu -x -p no:cacheprovider -s -k "c3m_fused or pair_pass" > gpurun_out/g10_tests.log 2>&1
tail -15 gpurun_out/g10_tests.log
for impl in 2 4 3; do timeout -s KILL 300 python tools/prof_pass.py C3 8 $impl split 2>&1 | tail -1; done > gpurun_out/g10_timing.txt
cat gpurun_out/g10_timing.txt
