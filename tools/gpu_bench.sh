mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/b_c3.log 2>&1
timeout 300 python bench.py --impl reference > gpurun_out/b_ref.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"xw_tma|xty_tc|reduce|prep_w|chol|vec_gram|apply|ritz|split" --log-file gpurun_out/b_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"xw_tma|xty_tc" -s 4 -c 2 -o gpurun_out/b_prof python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1
cat gpurun_out/b_c3.log gpurun_out/b_ref.log
