python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"ritz_values|chol_inv" -s 3 -c 2 -o gpurun_out/p7 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1
echo done
