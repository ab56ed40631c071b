mkdir -p gpurun_out
( timeout 120 ./tools/membench2 ; timeout 120 ./tools/membench ) > gpurun_out/e1_membench.log 2>&1
for d in 0 1 2 3; do PPCA_DBG=$d timeout 300 python tools/dbg_ka.py $d; done > gpurun_out/e1_dbg.log 2>&1
timeout 300 python tools/prof_pass.py C3 5 > gpurun_out/e1_prof.log 2>&1
cat gpurun_out/e1_membench.log gpurun_out/e1_dbg.log gpurun_out/e1_prof.log
