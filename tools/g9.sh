# round-2 re-entry check: full GPU suite, smoke, default bench line (C3 + also.C5), launch lists
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g9_smi.txt
timeout -s KILL 2400 python -m pytest tests -q -m gpu --durations=25 -p no:cacheprovider > gpurun_out/g9_tests.log 2>&1
tail -40 gpurun_out/g9_tests.log
timeout -s KILL 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g9_smoke.log 2>&1; tail -3 gpurun_out/g9_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/g9_bench.log 2>&1; tail -1 gpurun_out/g9_bench.log > gpurun_out/g9_bench.jsonl; cut -c1-600 gpurun_out/g9_bench.jsonl
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g9_c3_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1
python tools/launches.py gpurun_out/g9_c3_launches.csv > gpurun_out/g9_c3_launches.txt; head -30 gpurun_out/g9_c3_launches.txt
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g9_c5_launches.csv python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/g9_c5_launches.csv > gpurun_out/g9_c5_launches.txt; head -30 gpurun_out/g9_c5_launches.txt
