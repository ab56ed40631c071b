# round-1 final measurements: tests, bench lines, ncu launch list + full capture of the dominant kernel
mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -q -m gpu > gpurun_out/f_tests.log 2>&1; tail -3 gpurun_out/f_tests.log
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1; tail -1 gpurun_out/f_smoke.log
timeout -s KILL 600 python bench.py > gpurun_out/f_c3.log 2>&1; tail -1 gpurun_out/f_c3.log > gpurun_out/f_c3.jsonl
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/f_ref.log 2>&1; tail -1 gpurun_out/f_ref.log > gpurun_out/f_ref.jsonl
timeout -s KILL 900 python bench.py --config C5 > gpurun_out/f_c5.log 2>&1; tail -1 gpurun_out/f_c5.log > gpurun_out/f_c5.jsonl
timeout -s KILL 600 python bench.py --config C2 > gpurun_out/f_c2.log 2>&1; tail -1 gpurun_out/f_c2.log > gpurun_out/f_c2.jsonl
timeout -s KILL 900 python bench.py --config C4 > gpurun_out/f_c4.log 2>&1; tail -1 gpurun_out/f_c4.log > gpurun_out/f_c4.jsonl
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 3 --warmup 3 > /dev/null 2>&1
python tools/launches.py gpurun_out/f_launches.csv > gpurun_out/f_launches.txt
timeout -s KILL 1200 ncu --set full --import-source on --clock-control none -k regex:xwz_fused -c 1 -o gpurun_out/f_fused python bench.py --steps 2 --warmup 3 --no-cpu --no-lces > /dev/null 2>&1
ls -la gpurun_out/f_*
