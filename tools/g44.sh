mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "eigengame or c4 or C4 or huge or minibatch or table" > gpurun_out/g44_tests.log 2>&1; tail -3 gpurun_out/g44_tests.log
PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so AB_TAG=eg timeout -s KILL 400 python tools/ab_chain.py C4 2>&1 | grep -v Warn
PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so AB_TAG=eg timeout -s KILL 400 python tools/ab_chain.py C4 2>&1 | grep -v Warn
