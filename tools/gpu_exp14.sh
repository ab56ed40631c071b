for cf in 0 4; do PPCA_FUSED_CFG=$cf timeout -s KILL 100 python tools/prof_pass.py C3 5 2 split 2>&1 | sed "s/^/cfg=$cf /"; done
timeout -s KILL 100 python tools/prof_pass.py C3 5 3 split 2>&1 | sed "s/^/2kernel /"
