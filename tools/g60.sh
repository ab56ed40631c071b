# same-box timeline A/B of the one-step / two-step Cholesky sweep; C4 and C2 step timelines
for v in 0 1 0 1; do PPCA_CHOL2=$v PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 200 python tools/timeline.py C3 6 1 > gpurun_out/tl60_c3_chol$v.log 2>&1
awk -v v=$v '/reduce_splits_f64/ && /s13/ {rs=$1+$2} /chol_inv_reg/ {printf "chol2=%s chol end-after-splits %.1f  ", v, $1+$2-rs} /apply_rows/ {printf "apply end %.1f\n", $1+$2-rs}' gpurun_out/tl60_c3_chol$v.log; grep period gpurun_out/tl60_c3_chol$v.log; done
timeout -s KILL 300 python tools/timeline.py C4 4 > gpurun_out/tl60_c4.log 2>&1
timeout -s KILL 300 python tools/timeline.py C2 4 > gpurun_out/tl60_c2.log 2>&1
