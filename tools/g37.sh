# cluster-occupancy cap for the pair kernels + PDL: A/B at step level, then the parity subset
mkdir -p gpurun_out
for v in 1 0 1; do PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so PPCA_PDL=$v AB_TAG="pdl=$v" timeout -s KILL 400 python tools/ab_chain.py C3 C4 C5 2>&1 | grep -v Warn; done
timeout -s KILL 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "power or refine or c3m or C5 or c5" > gpurun_out/g37_tests.log 2>&1; tail -3 gpurun_out/g37_tests.log
