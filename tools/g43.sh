for g in 148 96 64 48 32 24 16; do PPCA_OJA_GRID=$g PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so AB_TAG="grid=$g" timeout -s KILL 200 python tools/ab_chain.py C2 2>&1 | grep -v Warn; done
PPCA_OJA_CLK=1 PPCA_OJA_GRID=148 PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 200 python tools/ab_chain.py C2 2>&1 | grep "step phases" | tail -1
PPCA_OJA_CLK=1 PPCA_OJA_GRID=32 PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 200 python tools/ab_chain.py C2 2>&1 | grep "step phases" | tail -1
