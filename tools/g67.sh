# C5 chain: two Gram slabs per SM (vec_gram_bal16), wider reduce_zp blocks: same-box timeline A/B, then the full GPU suite
mkdir -p gpurun_out
for cfg in "1 1" "2 4" "1 1" "2 4"; do set -- $cfg
PPCA_GRAM_CPSM=$1 PPCA_ZP_CPT=$2 PPCA_EXP_LIB=paper_2109_03709_b200/libppca_exp.so timeout -s KILL 300 python tools/timeline.py C5 4 1 > gpurun_out/tl67_$1_$2.log 2>&1
echo "gram_cpsm=$1 zp_cpt=$2: $(grep period gpurun_out/tl67_$1_$2.log)"
grep -E "reduce_zp_kernel|vec_gram_bal16|chol_inv_blk|apply_tiled" gpurun_out/tl67_$1_$2.log | sed -n 5,9p | cut -c1-110; done
timeout -s KILL 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s6b_tests.log 2>&1; tail -3 gpurun_out/s6b_tests.log
