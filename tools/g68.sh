# round-2 session-6 measurement set: smoke, bench lines (C3+C5 default, C4, C2, reference arm), ncu launch lists of the
# bench command (C3) and of a C5 run, ncu --set full of the pair kernel, timelines.  (The full GPU suite of the same
# tree ran in tools/g67.sh: profiles/r2_s6_gpu_tests.txt.)
mkdir -p gpurun_out
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s6_smoke.log 2>&1; tail -1 gpurun_out/s6_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/s6_bench.log 2>&1; tail -1 gpurun_out/s6_bench.log > gpurun_out/s6_bench.jsonl
timeout -s KILL 600 python bench.py --config C4 > gpurun_out/s6_c4.log 2>&1; tail -1 gpurun_out/s6_c4.log > gpurun_out/s6_c4.jsonl
timeout -s KILL 600 python bench.py --config C2 > gpurun_out/s6_c2.log 2>&1; tail -1 gpurun_out/s6_c2.log > gpurun_out/s6_c2.jsonl
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/s6_ref.log 2>&1; tail -1 gpurun_out/s6_ref.log > gpurun_out/s6_ref.jsonl
timeout -s KILL 300 python tools/timeline.py C3 6 1 > gpurun_out/s6_timeline_c3.txt 2>&1
timeout -s KILL 300 python tools/timeline.py C5 4 1 > gpurun_out/s6_timeline_c5.txt 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s6_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1
python tools/launches.py gpurun_out/s6_launches.csv > gpurun_out/s6_launches.txt 2>/dev/null
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s6_launches_c5.csv python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1
python tools/launches.py gpurun_out/s6_launches_c5.csv > gpurun_out/s6_launches_c5.txt 2>/dev/null
timeout -s KILL 1200 ncu --set full --import-source on --clock-control none -k regex:xwz_pair -c 1 -o gpurun_out/s6_pair python bench.py --steps 2 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:"vec_gram_bal16|apply_tiled|chol_inv_blk|reduce_zp_kernel" -c 8 -o gpurun_out/s6_c5chain python bench.py --config C5 --steps 2 --warmup 1 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1
rm -f gpurun_out/s6_launches.csv gpurun_out/s6_launches_c5.csv
ls -la gpurun_out/s6_*
cut -c1-400 gpurun_out/s6_bench.jsonl
