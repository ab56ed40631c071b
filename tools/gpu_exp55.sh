for cfg in 0 6 7; do echo "KR=64 cfg=$cfg"; PPCA_FUSED_CFG=$cfg timeout -s KILL 120 python tools/prof_pass.py C3 6 2 split 2>&1 | tail -1; done
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "C3s" 2>&1 | tail -1
