mkdir -p gpurun_out
python tools/ritz_clk.py 2>&1 | grep -v Warn
timeout -s KILL 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "power or refine or c5m or C5s or prop3 or theorem or stop or residual" > gpurun_out/g42_tests.log 2>&1; tail -3 gpurun_out/g42_tests.log
timeout -s KILL 200 python tools/sweep_nrg.py 2>&1 | grep nrg
PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so AB_TAG=ritz timeout -s KILL 400 python tools/ab_chain.py C3 C5 2>&1 | grep -v Warn
