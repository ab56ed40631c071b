# ysum_s with cp.async-staged loads and fp64 rows for the S tiles: C4 timeline, minibatch/EigenGame GPU tests, C4 bench line,
# ncu --set full of the C4 step kernels
mkdir -p gpurun_out
timeout -s KILL 300 python tools/timeline.py C4 6 1 > gpurun_out/s6_timeline_c4.txt 2>&1; tail -14 gpurun_out/s6_timeline_c4.txt | cut -c1-130
timeout -s KILL 1200 python -m pytest tests -x -q -m gpu -k "eigengame or c4 or huge_d or oja or window or minibatch or c2 or table" -p no:cacheprovider 2>&1 | tail -3
timeout -s KILL 600 python bench.py --config C4 > gpurun_out/s6_c4.log 2>&1; tail -1 gpurun_out/s6_c4.log > gpurun_out/s6_c4.jsonl; cut -c1-300 gpurun_out/s6_c4.jsonl
timeout -s KILL 900 ncu --set full --clock-control none -k regex:"eg_update|ysum_s|xty_tc|xw_tma" -s 40 -c 4 -o gpurun_out/s6_c4step python bench.py --config C4 --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1
ls -la gpurun_out/
