timeout -s KILL 300 python tools/ritz_clk.py
timeout -s KILL 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider --deselect tests/test_gpu_r2.py::test_huge_d_eigengame_and_refine_vs_oracle --deselect tests/test_gpu_r2.py::test_c5m_full_width_bf16_vs_oracle 2>&1 | tail -4
