mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/g21_san_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/g21_san_$tool.log
done
