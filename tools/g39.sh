for p in 1 0 1 0; do PPCA_PRIO=$p timeout -s KILL 200 python tools/sweep_nrg.py 2>&1 | grep nrg | sed "s/^/prio=$p /"; done
PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so PPCA_PRIO=1 AB_TAG=prio1 timeout -s KILL 400 python tools/ab_chain.py C3 C4 C5 2>&1 | grep -v Warn
PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so PPCA_PRIO=0 AB_TAG=prio0 timeout -s KILL 400 python tools/ab_chain.py C3 C4 C5 2>&1 | grep -v Warn
