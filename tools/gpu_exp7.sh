mkdir -p gpurun_out
timeout 300 python tools/prof_minibatch.py C2 200 > gpurun_out/e7.log 2>&1
timeout 300 python tools/prof_minibatch.py C4 50 >> gpurun_out/e7.log 2>&1
timeout 300 python tools/prof_pass.py C3 5 2 split >> gpurun_out/e7.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "power_priming or refine" 2>&1 | tail -2 >> gpurun_out/e7.log
python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e7_launches.csv python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1
cat gpurun_out/e7.log
