timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "power_priming" 2>&1 | grep -E "per-iteration|passed|failed|Error|error"
python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"ritz|chol" --log-file gpurun_out/e18.csv python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1
echo done
