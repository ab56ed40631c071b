mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -s > gpurun_out/g7_tests.log 2>&1
tail -3 gpurun_out/g7_tests.log
timeout -s KILL 900 python tools/huge_d.py --out gpurun_out/g7_huge_d.txt > gpurun_out/g7_huge_d.log 2>&1; tail -32 gpurun_out/g7_huge_d.log
timeout -s KILL 900 python bench.py --config C5 --no-cpu --no-e2e --no-lces > gpurun_out/g7_c5.log 2>&1; tail -1 gpurun_out/g7_c5.log | cut -c1-200
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g7_c5_launches.csv python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/g7_c5_launches.csv > gpurun_out/g7_c5_launches.txt
