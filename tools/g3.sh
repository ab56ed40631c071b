mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider -s > gpurun_out/g3_tests.log 2>&1
tail -3 gpurun_out/g3_tests.log
timeout -s KILL 600 python bench.py --no-cpu > gpurun_out/g3_c3.log 2>&1; tail -1 gpurun_out/g3_c3.log | cut -c1-400
timeout -s KILL 900 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/g3_c5.log 2>&1; tail -1 gpurun_out/g3_c5.log | cut -c1-400
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g3_c5_launches.csv python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/g3_c5_launches.csv > gpurun_out/g3_c5_launches.txt
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g3_c3_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/g3_c3_launches.csv > gpurun_out/g3_c3_launches.txt
