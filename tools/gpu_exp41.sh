timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "C5s or c5" -s 2>&1 | grep -E "parity|passed|failed|Error" | tail -12
timeout -s KILL 900 python -m pytest tests/test_full_size.py -x -q -m gpu -k "c5" -s 2>&1 | grep -E "parity|passed|failed|Error" | tail -5
timeout -s KILL 600 python tools/prof_pass.py C5 3 2 2>&1 | tail -1
timeout -s KILL 600 python bench.py --config C5 --no-cpu 2>&1 | tail -1
