timeout -s KILL 600 python bench.py --config C2 2>&1 | tail -1
timeout -s KILL 900 python bench.py --config C4 2>&1 | tail -1
