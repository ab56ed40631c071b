timeout -s KILL 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout -s KILL 300 python tools/prof_minibatch.py C4 20 split 2>&1 | tail -1
for rep in 1 2; do timeout -s KILL 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['roofline']['kernel_ms'], d['time_to_lces']['ms'])"; done
