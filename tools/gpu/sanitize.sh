# compute-sanitizer over the tiny workload (tools/sanitize_tiny.py); logs in gpurun_out/sanitize_*.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_tiny.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -4 gpurun_out/sanitize_$tool.log
done
