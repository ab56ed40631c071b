timeout -s KILL 300 python tools/prof_pass.py C5 2 2
timeout -s KILL 300 python tools/prof_pass.py C3 2 3 split
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "C5s or tcgen05-2kernel or eigengame or oja" 2>&1 | tail -1
