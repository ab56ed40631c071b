mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "power or refine or prop3 or theorem or c5m or C5s or residual or c3m or C1 or c1" > gpurun_out/g50_tests.log 2>&1; tail -3 gpurun_out/g50_tests.log
timeout -s KILL 900 python bench.py > gpurun_out/g50_bench.log 2>&1; tail -1 gpurun_out/g50_bench.log > gpurun_out/g50_bench.jsonl; python - <<'P'
import json
d=json.loads(open('gpurun_out/g50_bench.jsonl').read())
print('value', d['value'], 'ms', d['ms_per_step'], 'frac', d['roofline']['frac'], 'kernel_ms', d['roofline']['kernel_ms'], 'outside', d['step_outside_pass_ms'], 'ttl', d['time_to_lces'], 'clocks', d['clocks'])
c5=d['also']['C5']; print('C5', c5['value'], c5['ms_per_step'], c5['step_outside_pass_ms'], c5['time_to_lces']['ms'], c5['clocks'])
P
