mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_full_size.py -x -q -s 2>&1 | tail -15 > gpurun_out/e6_full.log
timeout 600 python bench.py --steps 10 --warmup 3 --config C5 --no-lces > gpurun_out/e6_c5.log 2>&1
timeout 300 python tools/prof_pass.py C5 3 2 >> gpurun_out/e6_c5.log 2>&1
cat gpurun_out/e6_full.log; cut -c1-1500 gpurun_out/e6_c5.log
