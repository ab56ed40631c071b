timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "eigengame or oja" 2>&1 | tail -1
timeout -s KILL 300 python tools/prof_minibatch.py C4 20 split 2>&1 | tail -1
