for n in 0 74 73 72 70 68 64; do PPCA_PAIR_NRG=$n timeout -s KILL 200 python tools/sweep_nrg.py 2>&1 | grep nrg; done
