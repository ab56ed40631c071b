# PDL for the chain kernels: parity subset, then step-level A/B (experiment build, PPCA_PDL=0/1)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "power or refine or eigengame or c3m or full" > gpurun_out/g36_tests.log 2>&1; tail -3 gpurun_out/g36_tests.log
for v in 0 1 0 1; do PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so PPCA_PDL=$v AB_TAG="pdl=$v" timeout -s KILL 300 python tools/ab_chain.py C3 C4 C2 2>&1 | grep -v Warn; done
