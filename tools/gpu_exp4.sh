mkdir -p gpurun_out
for d in 0 1 32; do PPCA_DBG=$d timeout 120 python tools/dbg_ka.py $d split 2>&1 | tail -1; done > gpurun_out/e4.log 2>&1
timeout 300 python tools/prof_pass.py C3 5 2 split >> gpurun_out/e4.log 2>&1
cat gpurun_out/e4.log
