timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "C5s" -s 2>&1 | grep -E "parity|passed|failed|Error|error" | tail -8
echo "---"
for pr in 0 1; do echo "pair=$pr"; PPCA_A2_PAIR=$pr timeout -s KILL 200 python tools/prof_pass.py C5 3 2 2>&1 | tail -1; done
timeout -s KILL 600 python -m pytest tests/test_full_size.py -x -q -m gpu -k "c5" -s 2>&1 | grep -E "parity|passed|failed|Error" | tail -3
