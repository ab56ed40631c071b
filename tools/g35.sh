# round-2 re-entry (session 4): full GPU suite, smoke, default bench line
mkdir -p gpurun_out
timeout -s KILL 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/g35_tests.log 2>&1; tail -5 gpurun_out/g35_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g35_smoke.log 2>&1; tail -1 gpurun_out/g35_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/g35_bench.log 2>&1; tail -1 gpurun_out/g35_bench.log
timeout -s KILL 300 python bench.py --config C4 > gpurun_out/g35_c4.log 2>&1; tail -1 gpurun_out/g35_c4.log
timeout -s KILL 300 python bench.py --config C2 > gpurun_out/g35_c2.log 2>&1; tail -1 gpurun_out/g35_c2.log
