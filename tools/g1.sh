mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout -s KILL 900 python bench.py --config C5 --no-cpu > gpurun_out/g1_c5.log 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g1_c5_launches.csv python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/g1_c5_launches.csv > gpurun_out/g1_c5_launches.txt
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g1_c3_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/g1_c3_launches.csv > gpurun_out/g1_c3_launches.txt
