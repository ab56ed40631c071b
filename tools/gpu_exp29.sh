set -x
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "oja" 2>&1 | tail -2
PPCA_OJA_CLK=1 timeout -s KILL 300 python tools/prof_minibatch.py C2 200 split 2>&1 | tail -3
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:oja_persistent -c 1 -o gpurun_out/oja_full python tools/prof_minibatch.py C2 20 split > gpurun_out/ncu_oja.log 2>&1
tail -3 gpurun_out/ncu_oja.log
