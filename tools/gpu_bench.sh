mkdir -p gpurun_out
timeout -s KILL 600 python bench.py > gpurun_out/b_c3.log 2>&1
timeout -s KILL 300 python bench.py --impl reference > gpurun_out/b_ref.log 2>&1
timeout -s KILL 600 python bench.py --config C5 --no-lces > gpurun_out/b_c5.log 2>&1
timeout -s KILL 300 python tools/prof_minibatch.py C4 30 split > gpurun_out/b_mb.log 2>&1
timeout -s KILL 300 python tools/prof_minibatch.py C2 200 split >> gpurun_out/b_mb.log 2>&1
timeout -s KILL 300 python tools/prof_pass.py C4 2 2 split >> gpurun_out/b_mb.log 2>&1
timeout -s KILL 300 python tools/prof_pass.py C3 5 2 split >> gpurun_out/b_mb.log 2>&1
timeout -s KILL 300 python tools/prof_pass.py C3 5 3 split >> gpurun_out/b_mb.log 2>&1
timeout -s KILL 300 python tools/prof_pass.py C5 2 2 >> gpurun_out/b_mb.log 2>&1
cat gpurun_out/b_mb.log
