mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "power_priming" 2>&1 | grep -E "parity|passed|failed|Error|error|assert" > gpurun_out/e11.log
timeout 120 python tools/prof_pass.py C3 5 2 split >> gpurun_out/e11.log 2>&1
timeout 120 python tools/prof_pass.py C3 5 3 split >> gpurun_out/e11.log 2>&1
cat gpurun_out/e11.log
