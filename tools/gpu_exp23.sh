timeout -s KILL 800 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"chol|ritz" --log-file gpurun_out/e23.csv python tools/prof_pass.py C3 3 2 split > /dev/null 2>&1
echo done
