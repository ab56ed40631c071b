export PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so
for rep in 1 2; do
for cfg in 0 1 5; do echo "cfg $cfg: $(PPCA_PAIR_CFG=$cfg timeout -s KILL 300 python tools/prof_pass.py C3 20 2 split 2>&1 | tail -1)"; done
echo "rowgroup: $(timeout -s KILL 300 python tools/prof_pass.py C3 20 4 split 2>&1 | tail -1)"
done
PPCA_PAIR_CFG=5 PPCA_TRACE=3 timeout -s KILL 300 python tools/prof_pass.py C3 4 2 split 2>&1 | tail -1; python tools/pair_trace.py | grep -v "^ *[0-9]"
