timeout -s KILL 900 python -m pytest tests/test_full_size.py -x -q -s 2>&1 | grep -E "parity|passed|failed|Error|assert" | tail -12
timeout -s KILL 800 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
