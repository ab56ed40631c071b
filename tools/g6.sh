mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_r2.py -q -m gpu -p no:cacheprovider -s -k "huge_d" > gpurun_out/g6_tests.log 2>&1
tail -5 gpurun_out/g6_tests.log
timeout -s KILL 900 python tools/huge_d.py --out gpurun_out/g6_huge_d.txt > gpurun_out/g6_huge_d.log 2>&1; tail -30 gpurun_out/g6_huge_d.log
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/g6_san_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/g6_san_$tool.log
done
