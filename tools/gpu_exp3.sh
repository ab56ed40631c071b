mkdir -p gpurun_out
for d in 0 2 3 7 32 35; do PPCA_DBG=$d timeout 120 python tools/dbg_ka.py $d 2>&1 | tail -1; done > gpurun_out/e3_dbg.log 2>&1
timeout 300 python tools/prof_pass.py C3 5 >> gpurun_out/e3_dbg.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -s -k "power_priming or refine" 2>&1 | grep -E "parity|passed|failed|Error" > gpurun_out/e3_parity.log
cat gpurun_out/e3_dbg.log gpurun_out/e3_parity.log
