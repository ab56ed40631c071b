timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "eigengame" -s 2>&1 | grep -E "parity|passed|failed|Error" | tail -8
timeout -s KILL 900 python -m pytest tests/test_full_size.py -x -q -m gpu -k "c4" -s 2>&1 | grep -E "parity|passed|failed|Error" | tail -4
timeout -s KILL 300 python tools/prof_minibatch.py C4 20 split 2>&1 | tail -1
PPCA_EG_MULTI=1 timeout -s KILL 300 python tools/prof_minibatch.py C4 20 split 2>&1 | tail -1
