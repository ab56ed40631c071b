timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:oja_persistent -c 1 -o gpurun_out/oja_full3 python tools/prof_minibatch.py C2 20 split > gpurun_out/ncu_oja.log 2>&1
tail -2 gpurun_out/ncu_oja.log
