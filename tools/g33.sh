timeout -s KILL 1200 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g33_huge.csv python tools/huge_d.py --steps 6 > /dev/null 2>&1
python tools/launches.py gpurun_out/g33_huge.csv | grep -v "store_raw\|house_\|colsum\|sqrt_lambda\|scale_kernel\|gamma\|init_rows\|planted" | head -20
