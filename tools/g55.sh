# pair kernel L2 policy sweep (experiment build): PPCA_PAIR_POL = hi | lo << 2 | re-read << 4 (0 last, 1 normal, 2 first, 3 unchanged)
for pol in 40 41 24 56 25 36 42 40; do
  echo "pol=$pol"; PPCA_PAIR_POL=$pol PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 120 python tools/l2_persist.py 0 0 2>&1 | grep step
done
