echo "current:"; python tools/ritz_clk.py 2>&1 | grep -v Warn | grep -v chol_inv
