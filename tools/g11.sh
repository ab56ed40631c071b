mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_r2.py -q -m gpu -p no:cacheprovider -s -k "c3m_fused or pair_pass" > gpurun_out/g11_tests.log 2>&1
grep -E "parity|passed|failed|Error" gpurun_out/g11_tests.log | tail -12
for cfg in 0 1 2 3; do echo "cfg $cfg: $(PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so PPCA_PAIR_CFG=$cfg timeout -s KILL 300 python tools/prof_pass.py C3 8 2 split 2>&1 | tail -1)"; done
echo "rowgroup: $(timeout -s KILL 300 python tools/prof_pass.py C3 8 4 split 2>&1 | tail -1)"
