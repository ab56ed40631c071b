mkdir -p gpurun_out
timeout -s KILL 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g45_c4.csv python tools/prof_minibatch.py C4 10 split > /dev/null 2>&1
python tools/launches.py gpurun_out/g45_c4.csv | head -12
timeout -s KILL 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g45_c3.csv python tools/sweep_nrg.py > /dev/null 2>&1
python tools/launches.py gpurun_out/g45_c3.csv | head -16
