# session 6, second half: Gram b-load rotation (no bank conflicts), fp64-staged IN in apply_tiled / vec_gram_generic:
# C5 timeline, full GPU suite, then the measurement set again (tools/g68.sh)
mkdir -p gpurun_out
timeout -s KILL 300 python tools/timeline.py C5 4 1 > gpurun_out/tl69_c5.log 2>&1; grep period gpurun_out/tl69_c5.log
timeout -s KILL 300 python tools/timeline.py C3 4 0 refine > gpurun_out/s6_timeline_c3_refine.txt 2>&1; tail -25 gpurun_out/s6_timeline_c3_refine.txt | cut -c1-120
grep -E "reduce_zp_kernel|vec_gram_bal16|chol_inv_blk|apply_tiled" gpurun_out/tl69_c5.log | sed -n 5,9p | cut -c1-110
timeout -s KILL 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/s6c_tests.log 2>&1; tail -3 gpurun_out/s6c_tests.log
bash tools/g68.sh
