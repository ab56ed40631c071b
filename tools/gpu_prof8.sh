python tools/prof_pass.py C5 1 2 > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:"xw_tma" -s 1 -c 1 -o gpurun_out/p8_c5 python tools/prof_pass.py C5 1 2 > /dev/null 2>&1
echo done
