timeout -s KILL 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout -s KILL 300 python bench.py 2>&1 | tail -1
timeout -s KILL 300 python tools/ritz_clk.py 2>&1 | tail -2
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python bench.py --steps 3 --warmup 3 --no-lces --no-cpu > /dev/null 2>&1
python tools/launches.py gpurun_out/c3_launches.csv | head -20
