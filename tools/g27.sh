mkdir -p gpurun_out
timeout -s KILL 300 python tools/ritz_clk.py
timeout -s KILL 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/g27_tests.log 2>&1; tail -3 gpurun_out/g27_tests.log
timeout -s KILL 900 python bench.py > gpurun_out/g27_bench.log 2>&1; tail -1 gpurun_out/g27_bench.log > gpurun_out/g27_bench.jsonl
timeout -s KILL 900 python bench.py --config C4 --no-cpu > gpurun_out/g27_c4.log 2>&1; tail -1 gpurun_out/g27_c4.log > gpurun_out/g27_c4.jsonl
timeout -s KILL 900 python bench.py --config C2 --no-cpu > gpurun_out/g27_c2.log 2>&1; tail -1 gpurun_out/g27_c2.log > gpurun_out/g27_c2.jsonl
python - <<'PY'
import json
for f in ["g27_bench","g27_c4","g27_c2"]:
    try:
        d=json.load(open(f"gpurun_out/{f}.jsonl")); print(f, d["ms_per_step"], d["value"], d.get("roofline",{}).get("frac"), json.dumps(d.get("time_to_lces"))[:300])
    except Exception as e: print(f, "ERR", e)
PY
