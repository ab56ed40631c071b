export PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit,clocks_event_reasons.active --format=csv
PPCA_PAIR_CFG=0 PPCA_TRACE=3 timeout -s KILL 300 python tools/prof_pass.py C3 4 2 split 2>&1 | tail -1; python tools/pair_trace.py | grep "median\|period\|clock"
(for k in $(seq 1 40); do nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader; sleep 0.05; done) > gpurun_out/g17_smi.txt &
timeout -s KILL 300 python tools/prof_pass.py C3 60 2 split 2>&1 | tail -1
wait; sort gpurun_out/g17_smi.txt | uniq -c | sort -rn | head
