mkdir -p gpurun_out
python tools/ritz_clk.py 2>&1 | grep -v Warn
timeout -s KILL 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/g48_tests.log 2>&1; tail -4 gpurun_out/g48_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g48_smoke.log 2>&1; tail -1 gpurun_out/g48_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/g48_bench.log 2>&1; tail -1 gpurun_out/g48_bench.log | cut -c1-600
