mkdir -p gpurun_out
PPCA_EG_CLK=1 PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 300 python tools/prof_minibatch.py C4 5 split > gpurun_out/g47.log 2>&1; grep -v Warn gpurun_out/g47.log | tail -3
PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so AB_TAG=eg2 timeout -s KILL 400 python tools/ab_chain.py C4 2>&1 | grep -v Warn
timeout -s KILL 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "eigengame or c4 or C4 or huge" > gpurun_out/g47_tests.log 2>&1; tail -3 gpurun_out/g47_tests.log
