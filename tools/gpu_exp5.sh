mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "parity|passed|failed|Error|error|assert" > gpurun_out/e5.log
timeout 300 python tools/prof_pass.py C3 5 2 split >> gpurun_out/e5.log 2>&1
python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e5_launches.csv python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e >> gpurun_out/e5.log 2>&1
cat gpurun_out/e5.log
