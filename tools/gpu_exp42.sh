timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4r_launches.csv python tools/prof_refine_c4.py > /dev/null 2>&1
python tools/launches.py gpurun_out/c4r_launches.csv | head -30
