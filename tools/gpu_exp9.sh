mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/e9.log
python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"chol|ritz|apply|vec_gram" --log-file gpurun_out/e9_launches.csv python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1
timeout 600 python bench.py --no-cpu --no-e2e >> gpurun_out/e9.log 2>&1
cat gpurun_out/e9.log | cut -c1-300
