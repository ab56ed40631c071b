for dbg in 0 1 2 4 6 8 14; do echo "dbg=$dbg"; PPCA_DBG=$dbg timeout -s KILL 300 python tools/prof_pass.py C3 6 2 split 2>&1 | tail -1; done
