mkdir -p gpurun_out
for d in 0 1 2 3 4 6 7 8 10 16 26; do PPCA_DBG=$d timeout 120 python tools/dbg_ka.py $d 2>&1 | tail -1; done > gpurun_out/e2_dbg.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -s -k "power_priming" 2>&1 | grep -E "parity|passed|failed" > gpurun_out/e2_parity.log
cat gpurun_out/e2_dbg.log gpurun_out/e2_parity.log
