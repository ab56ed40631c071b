timeout -s KILL 300 python tools/ritz_clk.py
timeout -s KILL 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "refine or parity or prop3 or theorem or c3m or c4m or C2 or ritz or full_basis" --deselect tests/test_gpu_r2.py::test_huge_d_eigengame_and_refine_vs_oracle --deselect tests/test_gpu_r2.py::test_c5m_full_width_bf16_vs_oracle 2>&1 | tail -3
