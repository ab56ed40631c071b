mkdir -p gpurun_out
python tools/prof_pass.py C3 3 2 split > gpurun_out/p2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p2_launches.csv python tools/prof_pass.py C3 3 2 split > gpurun_out/p2_ncu1.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:"xw_tma|xty_tc" -s 2 -c 2 -o gpurun_out/prof_c3split python tools/prof_pass.py C3 3 2 split > gpurun_out/p2_ncu2.log 2>&1
cat gpurun_out/p2_plain.log; tail -2 gpurun_out/p2_ncu2.log
