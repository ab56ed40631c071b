mkdir -p gpurun_out
export PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so
for cfg in 0 1; do PPCA_PAIR_CFG=$cfg PPCA_TRACE=3 timeout -s KILL 300 python tools/prof_pass.py C3 4 2 split 2>&1 | tail -1; python tools/pair_trace.py; done
