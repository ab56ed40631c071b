timeout -s KILL 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for rep in 1 2; do timeout -s KILL 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['pass']['ms'], d['time_to_lces'])"; done
timeout -s KILL 600 python bench.py --config C5 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['pass']['ms'])"
