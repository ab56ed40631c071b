mkdir -p gpurun_out
timeout -s KILL 300 python tools/prof_minibatch.py C4 50 split
timeout -s KILL 300 python tools/prof_minibatch.py C2 400 split
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g22_c4.csv python tools/prof_minibatch.py C4 10 split > /dev/null 2>&1
python tools/launches.py gpurun_out/g22_c4.csv | grep -v "planted\|gauss\|colsum\|mgs_step\|split_rows\|gamma\|qt_finish\|init_rows\|scale_rows\|row_norm\|planted_mean" | head -20
