# ncu --set full of the minibatch step kernels (C4 EigenGame, C2 Oja) and of the C3 chain / Ritz kernels
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:"eg_update|ysum_s|xty_tc|xw_tma|prep" -s 40 -c 10 -o gpurun_out/s6_c4step python bench.py --config C4 --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > gpurun_out/s6_c4step.log 2>&1; tail -2 gpurun_out/s6_c4step.log | cut -c1-200
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:"reduce_zp_gram|chol_inv_regt|apply_rows|ritz_values|reduce_splits" -s 10 -c 8 -o gpurun_out/s6_c3chain python bench.py --steps 2 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > gpurun_out/s6_c3chain.log 2>&1; tail -2 gpurun_out/s6_c3chain.log | cut -c1-200
ls -la gpurun_out/*.ncu-rep
