set -x
timeout 300 python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1; tail -1 gpurun_out/san_plain.log
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.log
done
