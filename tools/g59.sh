# two-step Cholesky sweep: bitwise check against the one-step sweep, step A/B, timeline
for v in 0 1; do PPCA_CHOL2=$v PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 200 python tools/chol2_bitwise.py 2>&1 | grep sha1; done
for v in 0 1 0 1; do PPCA_CHOL2=$v AB_TAG="chol2=$v" PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 300 python tools/ab_chain.py C3 2>&1 | grep step; done
timeout -s KILL 200 python tools/timeline.py C3 5 1 > gpurun_out/tl59_c3.log 2>&1
sed -n 3,16p gpurun_out/tl59_c3.log
