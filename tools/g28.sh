export PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so
for dbg in 0 32 1 33; do echo "DBG=$dbg $(PPCA_DBG=$dbg timeout -s KILL 300 python tools/prof_pass.py C5 2 2 2>&1 | tail -1)"; done
timeout -s KILL 900 python -m pytest tests/test_full_size.py -q -m gpu -p no:cacheprovider -s -k "c3_full_size_power_and_refine" 2>&1 | grep -E "parity|passed|failed|Error|assert" | head
