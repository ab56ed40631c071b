# reduce_zp_gram v2 (2 features per CTA, cluster row gather) + operand split fused into CholQR's apply
timeout -s KILL 200 python tools/timeline.py C3 5 1 > gpurun_out/tl58_c3.log 2>&1
timeout -s KILL 300 python tools/ab_chain.py C3 > gpurun_out/ab58.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py tests/test_full_size.py -x -q -m gpu > gpurun_out/t58.log 2>&1
