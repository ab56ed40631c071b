python tools/prof_pass.py C3 2 2 split > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"chol_inv" -s 2 -c 1 -o gpurun_out/p6_chol python tools/prof_pass.py C3 2 2 split > /dev/null 2>&1
echo done
