mkdir -p gpurun_out
python tools/prof_minibatch.py C4 20 split > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"xw_tma|xty_tc|ysum|tn_kernel|reduce|eg_|apply|prep_w|row_norm|scale_rows" -s 70 -c 60 --log-file gpurun_out/p3_launches.csv python tools/prof_minibatch.py C4 20 split > /dev/null 2>&1
echo done
