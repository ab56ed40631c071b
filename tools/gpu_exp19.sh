timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "power_priming or refine" 2>&1 | tail -1
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"ritz|chol|xwz" --log-file gpurun_out/e19.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1
timeout -s KILL 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-250
