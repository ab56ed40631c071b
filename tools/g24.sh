timeout -s KILL 300 python tools/prof_minibatch.py C4 50 split
timeout -s KILL 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "c4 or C4 or oja or eigengame or C2" 2>&1 | tail -2
timeout -s KILL 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g24_c4.csv python tools/prof_minibatch.py C4 10 split > /dev/null 2>&1
python tools/launches.py gpurun_out/g24_c4.csv | grep "ppca::" | head -12
