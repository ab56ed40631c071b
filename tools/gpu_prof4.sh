mkdir -p gpurun_out
python tools/prof_pass.py C3 3 2 split > gpurun_out/p4_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"xwz_fused|xw_tma" -s 1 -c 2 -o gpurun_out/prof_fused python tools/prof_pass.py C3 3 2 split > gpurun_out/p4_ncu.log 2>&1
tail -2 gpurun_out/p4_ncu.log
