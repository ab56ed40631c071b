mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "c5m or C5s or c5s or huge" > gpurun_out/g40_tests.log 2>&1; tail -3 gpurun_out/g40_tests.log
for v in 1 0; do PPCA_KB_WIDE=$v PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so AB_TAG="wide=$v" timeout -s KILL 400 python tools/ab_chain.py C5 2>&1 | grep -v Warn; done
