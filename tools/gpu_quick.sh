# quick GPU check: full GPU test suite (parity printed) + C3 pass timing (fp32 and split)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "parity|passed|failed|Error|error|assert" > gpurun_out/q_pytest.log; echo "pytest done" >> gpurun_out/q_pytest.log
timeout 300 python tools/prof_pass.py C3 5 2 > gpurun_out/q_prof.log 2>&1
timeout 300 python tools/prof_pass.py C3 5 2 split >> gpurun_out/q_prof.log 2>&1
cat gpurun_out/q_pytest.log gpurun_out/q_prof.log
