mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/e10.log
timeout 600 python bench.py --no-cpu >> gpurun_out/e10.log 2>&1
cat gpurun_out/e10.log
