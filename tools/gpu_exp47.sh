for lag in 0 1 2 3; do echo "lag=$lag"; PPCA_FUSED_LAG=$lag timeout -s KILL 120 python tools/prof_pass.py C3 6 2 split 2>&1 | tail -1; done
