# EigenGame update writing the next window pass's operand split: bitwise check, step A/B, EigenGame GPU tests
for v in 0 1; do PPCA_EG_PREP=$v PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 300 python tools/egprep_bitwise.py 2>&1 | grep sha1; done
for v in 0 1 0 1; do PPCA_EG_PREP=$v AB_TAG="egprep=$v" PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 300 python tools/ab_chain.py C4 2>&1 | grep -i "step"; done
timeout -s KILL 900 python -m pytest tests -x -q -m gpu -k "eigengame or c4 or huge_d" -p no:cacheprovider 2>&1 | tail -3
