PPCA_EG_CLK=1 PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 300 python tools/prof_minibatch.py C4 5 split > gpurun_out/g46.log 2>&1; grep -v Warn gpurun_out/g46.log | tail -5
