timeout -s KILL 300 python tools/prof_minibatch.py C4 20 split 2>&1 | tail -1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/prof_minibatch.py C4 10 split > /dev/null 2>&1
python tools/launches.py gpurun_out/c4_launches.csv | head -30
