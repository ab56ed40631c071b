mkdir -p gpurun_out
timeout -s KILL 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/g20_tests.log 2>&1; tail -3 gpurun_out/g20_tests.log
timeout -s KILL 900 python bench.py > gpurun_out/g20_bench.log 2>&1; tail -1 gpurun_out/g20_bench.log > gpurun_out/g20_bench.jsonl; cut -c1-300 gpurun_out/g20_bench.jsonl
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g20_c3_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1
python tools/launches.py gpurun_out/g20_c3_launches.csv > gpurun_out/g20_c3_launches.txt; head -14 gpurun_out/g20_c3_launches.txt
timeout -s KILL 1200 ncu --set full --import-source on --clock-control none -k regex:xwz_pair -c 1 -o gpurun_out/g20_pair python bench.py --steps 2 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1; ls -la gpurun_out/g20_pair*
