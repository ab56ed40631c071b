# final tree of round 2: full GPU suite + smoke
mkdir -p gpurun_out
timeout -s KILL 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s6d_tests.log 2>&1; tail -3 gpurun_out/s6d_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s6d_smoke.log 2>&1; tail -2 gpurun_out/s6d_smoke.log
