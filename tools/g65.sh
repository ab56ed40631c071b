# register-tiled Cholesky sweep (chol_inv_sweep2t): bitwise vs the packed two-step sweep, same-box timeline A/B
mkdir -p gpurun_out
for v in 2 3 4 5 6; do PPCA_CHOL2=$v PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 200 python tools/chol2_bitwise.py 2>&1 | grep -E "sha1|rror"; done
for v in 2 3 4 5 6 2 3 4 5 6; do
PPCA_CHOL2=$v PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 200 python tools/timeline.py C3 6 1 > gpurun_out/tl65.log 2>&1
awk -v v="$v" '/reduce_splits_f64/ && /s13/ {rs=$1+$2} /chol_inv_reg/ {printf "chol2=%s chol end-after-splits %.1f  ", v, $1+$2-rs} /apply_rows/ {printf "apply end %.1f\n", $1+$2-rs}' gpurun_out/tl65.log | tail -3; grep period gpurun_out/tl65.log; done
