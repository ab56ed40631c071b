mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_r2.py -q -m gpu -p no:cacheprovider -s -k "distributed or one_rank or huge" > gpurun_out/g8_tests.log 2>&1
tail -3 gpurun_out/g8_tests.log
timeout -s KILL 900 python tools/huge_d.py --out gpurun_out/g8_huge_d.txt > gpurun_out/g8_huge_d.log 2>&1; grep "ms\|gbs" gpurun_out/g8_huge_d.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g8_huge_launches.csv python tools/huge_d.py --steps 8 > /dev/null 2>&1
python tools/launches.py gpurun_out/g8_huge_launches.csv > gpurun_out/g8_huge_launches.txt; head -25 gpurun_out/g8_huge_launches.txt
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g8_c4_launches.csv python bench.py --config C4 --steps 2 --warmup 3 --no-cpu --no-lces > /dev/null 2>&1
python tools/launches.py gpurun_out/g8_c4_launches.csv > gpurun_out/g8_c4_launches.txt; head -25 gpurun_out/g8_c4_launches.txt
