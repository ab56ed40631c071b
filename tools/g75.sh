# ncu --set full of the C3 chain kernels (one launch each) and the Ritz values kernel
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none -k regex:"reduce_zp_gram|chol_inv_regt|apply_rows|ritz_values" -s 8 -c 4 -o gpurun_out/s6_c3chain python bench.py --steps 2 --warmup 3 --no-cpu --no-lces --no-e2e --no-extra > gpurun_out/s6_c3chain.log 2>&1; tail -1 gpurun_out/s6_c3chain.log | cut -c1-200
ls -la gpurun_out/
