timeout -s KILL 100 python tools/prof_pass.py C3 5 2 split 2>&1 | sed "s/^/fused /"
timeout -s KILL 100 python tools/prof_pass.py C3 5 3 split 2>&1 | sed "s/^/2k /"
