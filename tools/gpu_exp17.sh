timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"chol|ritz|apply|vec_gram" --log-file gpurun_out/e17.csv python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1
timeout -s KILL 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-300
