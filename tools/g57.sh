# reduce_zp_gram (Z reduction + CholQR Gram in one cluster launch): timeline, step A/B, power-path GPU tests
timeout -s KILL 200 python tools/timeline.py C3 5 1 > gpurun_out/tl57_c3.log 2>&1
timeout -s KILL 300 python tools/ab_chain.py C3 > gpurun_out/ab57.log 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/t57.log 2>&1
