for v in 1 0 1 0; do PPCA_KEEPX=$v PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so AB_TAG="keepx=$v" timeout -s KILL 400 python tools/ab_chain.py C4 2>&1 | grep -v Warn; done
