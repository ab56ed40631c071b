mkdir -p gpurun_out
for pf in 0 2 4 8 16; do PPCA_FUSED_PF=$pf timeout 120 python tools/prof_pass.py C3 5 2 split 2>&1 | sed "s/^/pf=$pf /"; done > gpurun_out/e12.log
cat gpurun_out/e12.log
