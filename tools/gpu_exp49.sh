for rep in 1 2; do
for lag in 0 2; do echo "lag=$lag"; PPCA_FUSED_LAG=$lag timeout -s KILL 300 python bench.py --no-cpu --no-lces --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['pass']['ms'])"; done
done
