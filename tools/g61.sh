# packed two-step Cholesky sweep: bitwise vs one-step, same-box timeline A/B (variant 1 vs 2, CQ 8 / 16)
for v in 0 2; do PPCA_CHOL2=$v PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 200 python tools/chol2_bitwise.py 2>&1 | grep sha1; done
for cfg in "1 8" "2 8" "2 16" "1 8" "2 8" "2 16"; do set -- $cfg
PPCA_CHOL2=$1 PPCA_CHOL_CQ=$2 PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 200 python tools/timeline.py C3 6 1 > gpurun_out/tl61.log 2>&1
awk -v v="$1/$2" '/reduce_splits_f64/ && /s13/ {rs=$1+$2} /chol_inv_reg/ {printf "chol2/cq=%s chol end-after-splits %.1f  ", v, $1+$2-rs} /apply_rows/ {printf "apply end %.1f\n", $1+$2-rs}' gpurun_out/tl61.log | tail -3; grep period gpurun_out/tl61.log; done
