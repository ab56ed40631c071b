timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "eigengame or oja" -s 2>&1 | grep -E "parity|passed|failed|Error" | tail -12
timeout -s KILL 900 python -m pytest tests/test_full_size.py -x -q -m gpu -k "c4 or c2" -s 2>&1 | grep -E "parity|passed|failed|Error" | tail -4
timeout -s KILL 300 python tools/prof_minibatch.py C4 20 split 2>&1 | tail -1
