# ritz_values_kernel opt bits: phase clocks and agreement of theta / E with the baseline kernel (same box)
for o in 0 1 2 4 7; do PPCA_RITZ_OPT=$o PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 300 python tools/ritz_opt_ab.py 2>&1 | grep -E "opt=|rror|Trace" ; done
python tools/ritz_opt_ab.py cmp 0 1 2 4 7
for o in 0 7 0 7; do PPCA_RITZ_OPT=$o AB_TAG="ritz_opt=$o" PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 300 python tools/refine_ab.py 4 2>&1 | tail -2; done
# product library with the tiled sweep as the default (power step, C5's blocked Cholesky, Ritz kernels)
timeout -s KILL 900 python -m pytest tests -x -q -m gpu -k "c3m or c5m or c5s or c1 or ritz or stop_rule or orthonormal_flag or smoke" -p no:cacheprovider 2>&1 | tail -3
timeout -s KILL 300 python tools/timeline.py C5 4 1 > gpurun_out/s6_timeline_c5.txt 2>&1; grep -E "period|chol_inv" gpurun_out/s6_timeline_c5.txt | head -8
