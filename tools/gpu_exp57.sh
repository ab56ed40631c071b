for lag in 2 0 3; do echo "lag=$lag"; PPCA_FUSED_LAG=$lag timeout -s KILL 300 python bench.py --no-cpu --no-lces --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"; done
timeout -s KILL 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
