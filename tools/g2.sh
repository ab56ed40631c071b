mkdir -p gpurun_out
timeout -s KILL 2400 python -m pytest tests -q -m gpu --durations=20 -p no:cacheprovider > gpurun_out/g2_tests.log 2>&1
tail -40 gpurun_out/g2_tests.log
