for v in nws4 nws3 nws6 nws4; do cp abtest/lib_$v.so paper_2109_03709_b200/libppca.so; echo "$v"; timeout -s KILL 200 python tools/prof_pass.py C5 3 2 2>&1 | tail -1; done
