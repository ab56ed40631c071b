mkdir -p gpurun_out
export PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so
PPCA_PAIR_CFG=1 timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:xwz_pair -c 1 -o gpurun_out/g12_pair python tools/prof_pass.py C3 2 2 split > gpurun_out/g12_ncu.log 2>&1
tail -3 gpurun_out/g12_ncu.log
ls -la gpurun_out/
