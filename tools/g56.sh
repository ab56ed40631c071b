# live timeline of the C3 step (CUPTI via torch.profiler) + refine Ritz-solver A/B (experiment build)
timeout -s KILL 200 python tools/timeline.py C3 5 1 > gpurun_out/tl_c3.log 2>&1
timeout -s KILL 200 python tools/timeline.py C3 5 0 > gpurun_out/tl_c3_nohist.log 2>&1
for j in 0 1 0 1; do PPCA_RITZ_JACOBI=$j PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 200 python tools/refine_ab.py 4 10 2>&1 | grep refine_ex; done
