ncu --set full --clock-control none --import-source on -k regex:k_part_dedup --launch-skip 5 --launch-count 1 -o gpurun_out/prof_part_dedup -f python tools/sampler_bench.py --config papers --reps 0 --paths part > /dev/null 2> gpurun_out/ncu_part_dedup.err
tail -2 gpurun_out/ncu_part_dedup.err
ncu --set full --clock-control none --import-source on -k regex:k_part_tile --launch-skip 11 --launch-count 1 -o gpurun_out/prof_part_tile1 -f python tools/sampler_bench.py --config papers --reps 0 --paths part > /dev/null 2>> gpurun_out/ncu_part_dedup.err
bash tools/gpu/sanitize.sh
