set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "oja" -s 2>&1 | grep -E "parity|passed|failed|Error|error" | tail -20
timeout -s KILL 900 python -m pytest tests/test_full_size.py -x -q -m gpu -k "c2" -s 2>&1 | grep -E "parity|passed|failed|Error|error" | tail -8
timeout -s KILL 600 python bench.py --config C2 2>&1 | tail -1
