for v in 0 1 2 0; do PPCA_A2P_VAR=$v PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so AB_TAG="a2var=$v" timeout -s KILL 300 python tools/ab_chain.py C5 2>&1 | grep "kernel A"; done
