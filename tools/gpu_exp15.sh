timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1
