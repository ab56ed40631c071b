export PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so
timeout -s KILL 900 python -m pytest tests/test_gpu_r2.py -q -m gpu -p no:cacheprovider -s -k "c3m_fused or pair_pass" > gpurun_out/g16_tests.log 2>&1
grep -E "parity\]|passed|failed" gpurun_out/g16_tests.log | tail -6
for cfg in 0 1 2 3 4; do echo "cfg $cfg"; PPCA_PAIR_CFG=$cfg PPCA_TRACE=3 timeout -s KILL 300 python tools/prof_pass.py C3 4 2 split 2>&1 | tail -1; python tools/pair_trace.py | grep "median\|period"; done
