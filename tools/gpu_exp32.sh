for dbg in 0 32; do
  echo "dbg=$dbg"; PPCA_OJA_DBG=$dbg timeout -s KILL 120 python tools/prof_minibatch.py C2 200 split 2>&1 | tail -1
done
