mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/b_c3.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --impl reference > gpurun_out/b_ref.log 2>&1
cat gpurun_out/b_c3.log gpurun_out/b_ref.log
