# round-2 session-5 measurement set: full GPU suite, smoke, bench lines (C3+C5 default, C4, C2, reference arm),
# ncu launch list of the bench command, ncu --set full of the pair kernel
mkdir -p gpurun_out
timeout -s KILL 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s5_tests.log 2>&1; tail -2 gpurun_out/s5_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s5_smoke.log 2>&1; tail -1 gpurun_out/s5_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/s5_bench.log 2>&1; tail -1 gpurun_out/s5_bench.log > gpurun_out/s5_bench.jsonl
timeout -s KILL 600 python bench.py --config C4 > gpurun_out/s5_c4.log 2>&1; tail -1 gpurun_out/s5_c4.log > gpurun_out/s5_c4.jsonl
timeout -s KILL 600 python bench.py --config C2 > gpurun_out/s5_c2.log 2>&1; tail -1 gpurun_out/s5_c2.log > gpurun_out/s5_c2.jsonl
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/s5_ref.log 2>&1; tail -1 gpurun_out/s5_ref.log > gpurun_out/s5_ref.jsonl
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1
python tools/launches.py gpurun_out/s5_launches.csv > gpurun_out/s5_launches.txt 2>/dev/null
timeout -s KILL 1200 ncu --set full --import-source on --clock-control none -k regex:xwz_pair -c 1 -o gpurun_out/s5_pair python bench.py --steps 2 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > /dev/null 2>&1
ls -la gpurun_out/s5_*
