mkdir -p gpurun_out
timeout -s KILL 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g23_c4.csv python tools/prof_minibatch.py C4 10 split > /dev/null 2>&1
python tools/launches.py gpurun_out/g23_c4.csv | grep -v "planted\|gauss\|colsum\|mgs_step\|split_rows\|gamma\|qt_finish\|init_rows\|scale_rows\|row_norm\|planted_mean" | head -12
timeout -s KILL 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g23_c3.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1
python tools/launches.py gpurun_out/g23_c3.csv | grep -v "planted\|gauss\|colsum\|mgs_step\|split_rows\|gamma\|qt_finish\|init_rows\|scale_rows\|row_norm\|planted_mean" | head -16
