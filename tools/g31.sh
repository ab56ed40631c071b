timeout -s KILL 300 python tools/ritz_clk.py
timeout -s KILL 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "refine or parity or prop3 or theorem or c3m or C2 or ritz or full_basis or c5m or stop_rule or certified" --deselect tests/test_gpu_r2.py::test_huge_d_eigengame_and_refine_vs_oracle 2>&1 | tail -3
timeout -s KILL 900 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none -k regex:ritz --csv --log-file gpurun_out/g31_c5.csv python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-lces --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/g31_c5.csv | head -3
