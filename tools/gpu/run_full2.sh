timeout 2400 python -X faulthandler -m pytest tests -m gpu -x -v -p no:cacheprovider > gpurun_out/r2_gputests_full_v.log 2>&1; echo rc=$?
grep -n "PASSED\|FAILED\|ERROR\|Fatal\|Segmentation\|Aborted" gpurun_out/r2_gputests_full_v.log | tail -15
grep -n -B5 -A30 "Fatal Python error" gpurun_out/r2_gputests_full_v.log | head -80
