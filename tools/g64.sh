# round-2 session-6 re-entry check: full GPU suite, smoke, default bench line (restored container, rebuilt .so)
mkdir -p gpurun_out
timeout -s KILL 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s6_tests.log 2>&1; tail -2 gpurun_out/s6_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s6_smoke.log 2>&1; tail -1 gpurun_out/s6_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/s6_bench.log 2>&1; tail -1 gpurun_out/s6_bench.log > gpurun_out/s6_bench.jsonl
timeout -s KILL 300 python tools/timeline.py C3 6 1 > gpurun_out/s6_timeline_c3.txt 2>&1
cut -c1-600 gpurun_out/s6_bench.jsonl
