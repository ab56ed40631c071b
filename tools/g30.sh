timeout -s KILL 900 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g30_c5.csv python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-lces --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/g30_c5.csv | grep -v "planted\|gauss\|colsum\|mgs_step\|split_rows\|gamma\|qt_finish\|init_rows\|scale_rows\|row_norm\|planted_mean\|store_raw\|house_\|sqrt_lambda\|scale_kernel" | head -20
timeout -s KILL 900 python bench.py --config C5 --no-cpu --no-e2e > gpurun_out/g30_c5.log 2>&1; tail -1 gpurun_out/g30_c5.log > gpurun_out/g30_c5.jsonl
python -c "
import json;d=json.load(open('gpurun_out/g30_c5.jsonl')); print(d['ms_per_step'], d['step_outside_pass_ms'], d['roofline']['pass'], d['roofline']['tensor_context'])"
