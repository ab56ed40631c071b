mkdir -p gpurun_out
timeout -s KILL 1200 python tools/huge_d.py --out gpurun_out/r2_huge_d.txt > gpurun_out/g32_huge_d.log 2>&1; echo "huge_d rc=$?"; tail -25 gpurun_out/g32_huge_d.log
timeout -s KILL 2400 python tools/table12_repro.py --seeds 10 --out gpurun_out/r2_table12_repro.txt > gpurun_out/g32_table12.log 2>&1; echo "table12 rc=$?"; tail -40 gpurun_out/g32_table12.log
