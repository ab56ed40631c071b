mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "parity|passed|failed|Error|error|assert" > gpurun_out/e8.log
timeout 300 python tools/prof_minibatch.py C2 200 split >> gpurun_out/e8.log 2>&1
timeout 300 python tools/prof_minibatch.py C4 50 split >> gpurun_out/e8.log 2>&1
timeout 300 python tools/prof_minibatch.py C4 50 >> gpurun_out/e8.log 2>&1
timeout 300 python tools/prof_pass.py C3 5 2 split >> gpurun_out/e8.log 2>&1
cat gpurun_out/e8.log
