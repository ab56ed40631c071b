export PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so
for dbg in 0 32 1 33; do PPCA_DBG=$dbg timeout -s KILL 300 python tools/ablate_a2.py C5 4 2>&1 | tail -1; done
