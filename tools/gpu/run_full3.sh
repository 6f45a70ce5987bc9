timeout 2400 python -X faulthandler -m pytest tests -m gpu -x -v -p no:cacheprovider > gpurun_out/r2_gputests_full_v.log 2>&1; echo rc=$?
grep -n "FAILED\|ERROR\|Fatal\|passed\|failed" gpurun_out/r2_gputests_full_v.log | tail -8
timeout 300 python tools/pcie_bidir.py 2>/dev/null | tail -1
DGNN_ASM_TRACE=1 timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_trace.json 2> gpurun_out/r2_bench_trace.err; grep "asm-trace" gpurun_out/r2_bench_trace.err
ncu --set full --clock-control none --import-source on -k regex:k_part_dedup --launch-skip 5 --launch-count 1 -o gpurun_out/prof_part_dedup3 -f python tools/sampler_bench.py --config papers --reps 0 --paths part > /dev/null 2>&1
