timeout -s KILL 800 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "refine Ritz|sampled|passed|failed|Error|assert" | tail -30
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"ritz|chol" --log-file gpurun_out/e24.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout -s KILL 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['time_to_lces'])"
