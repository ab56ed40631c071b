mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_r2.py -q -m gpu -p no:cacheprovider -s > gpurun_out/g5_tests.log 2>&1
tail -3 gpurun_out/g5_tests.log
timeout -s KILL 900 python bench.py > gpurun_out/g5_bench.log 2>&1; tail -1 gpurun_out/g5_bench.log | cut -c1-200
timeout -s KILL 1500 python tools/table12_repro.py --seeds 10 --out gpurun_out/g5_table12.txt > gpurun_out/g5_table12.log 2>&1
tail -30 gpurun_out/g5_table12.log
