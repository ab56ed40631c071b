timeout -s KILL 300 python tools/ritz_clk.py 2>&1 | tail -4
timeout -s KILL 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
