# quick GPU check: parity of the pass + C3 pass timing + bench line
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "power or refine" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 300 python tools/prof_pass.py C3 5 > gpurun_out/q_prof.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/q_bench.log 2>&1
tail -2 gpurun_out/q_pytest.log; cat gpurun_out/q_prof.log; cut -c1-400 gpurun_out/q_bench.log
