mkdir -p gpurun_out
PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so AB_TAG=ysum timeout -s KILL 400 python tools/ab_chain.py C4 2>&1 | grep -v Warn
timeout -s KILL 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "eigengame or c4 or C4 or huge or sampled or minibatch or oja" > gpurun_out/g53_tests.log 2>&1; tail -3 gpurun_out/g53_tests.log
timeout -s KILL 600 python bench.py --config C4 > gpurun_out/g53_c4.log 2>&1; tail -1 gpurun_out/g53_c4.log | cut -c1-400
