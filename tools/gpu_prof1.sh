set -x
mkdir -p gpurun_out
python tools/prof_pass.py C3 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/prof_pass.py C3 3 > gpurun_out/ncu1.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:"xw_tc|xty_tc" -s 2 -c 2 -o gpurun_out/prof_c3 python tools/prof_pass.py C3 3 > gpurun_out/ncu2.log 2>&1
echo done
