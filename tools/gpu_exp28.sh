set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "oja" -s 2>&1 | grep -E "parity|passed|failed|Error|error" | tail -20
PPCA_OJA_CLK=1 timeout -s KILL 300 python bench.py --config C2 --no-lces --no-cpu 2>&1 | grep -E "oja_persistent\]" | tail -3
timeout -s KILL 900 python -m pytest tests/test_full_size.py -x -q -m gpu -k "c2" -s 2>&1 | grep -E "parity|passed|failed|Error|error" | tail -8
timeout -s KILL 600 python bench.py --config C2 2>&1 | tail -1
