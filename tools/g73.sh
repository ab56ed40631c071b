# reduce_zp_gram with cp.async-staged loads: W bitwise (sha1 as in profiles/r2_s6_chol_tiles_ab.txt), C3 timeline, power-path
# GPU tests, default bench line, ncu launch list
mkdir -p gpurun_out
PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 200 python tools/chol2_bitwise.py 2>&1 | grep -E "sha1|rror"
timeout -s KILL 300 python tools/timeline.py C3 6 1 > gpurun_out/s6_timeline_c3.txt 2>&1; grep period gpurun_out/s6_timeline_c3.txt; sed -n 20,30p gpurun_out/s6_timeline_c3.txt | cut -c1-120
timeout -s KILL 1500 python -m pytest tests -x -q -m gpu -k "c3 or c1 or power or pair or nccl or orth or stop or smoke or resume" -p no:cacheprovider 2>&1 | tail -3
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout -s KILL 900 python bench.py > gpurun_out/s6_bench.log 2>&1; tail -1 gpurun_out/s6_bench.log > gpurun_out/s6_bench.jsonl; cut -c1-300 gpurun_out/s6_bench.jsonl
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s6_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1
python tools/launches.py gpurun_out/s6_launches.csv > gpurun_out/s6_launches.txt 2>/dev/null; rm -f gpurun_out/s6_launches.csv
