timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4m2.csv python tools/prof_minibatch.py C4 10 split > /dev/null 2>&1
python tools/launches.py gpurun_out/c4m2.csv | grep -v "planted\|mgs_step\|gauss\|colsum\|split_rows\|planted_mean\|gamma\|qt_finish" | head -14
