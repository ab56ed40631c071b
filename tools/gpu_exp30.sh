PPCA_OJA_CLK=1 timeout -s KILL 300 python tools/prof_minibatch.py C2 200 split 2>&1 | tail -3
