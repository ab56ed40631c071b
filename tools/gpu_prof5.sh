mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"xwz|xw_tma|xty_tc|reduce|prep_w|chol|vec_gram|apply|ritz" --log-file gpurun_out/p5_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"xwz" -s 2 -c 1 -o gpurun_out/p5_prof python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-lces > /dev/null 2>&1
echo done
