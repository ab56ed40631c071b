for d in 0 2; do for cf in 0 2; do PPCA_DBG=$d PPCA_FUSED_CFG=$cf timeout -s KILL 100 python tools/prof_pass.py C3 5 2 split 2>&1 | sed "s/^/dbg=$d cfg=$cf /"; done; done
