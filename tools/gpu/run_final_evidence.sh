bash tools/ncu_round2.sh
ls gpurun_out/prof_*_r2.ncu-rep
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_tiny.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -1 gpurun_out/sanitize_$tool.log
done
