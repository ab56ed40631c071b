timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "power_priming and C3s" 2>&1 | grep -E "parity|passed|failed|Error|error"
for d in 0 1; do PPCA_DBG=$d timeout -s KILL 100 python tools/prof_fused_dbg.py 2>&1 | tail -1; done
timeout -s KILL 100 python tools/prof_pass.py C3 5 2 split
