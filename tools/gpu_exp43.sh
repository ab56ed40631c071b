timeout -s KILL 600 python tools/prof_refine_c4.py 2>&1 | tail -5
timeout -s KILL 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout -s KILL 900 python bench.py --config C4 2>&1 | tail -1 > gpurun_out/bench_c4.jsonl
timeout -s KILL 300 python bench.py 2>&1 | tail -1 > gpurun_out/bench_c3.jsonl
