timeout 900 python -m pytest tests/test_gpu_sampler_paths.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/sampler_bench.py --config papers --reps 3 --out gpurun_out/sampler_papers3.json 2> gpurun_out/sampler_papers3.err | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_part|k_seed_sort|scan_kernel|k_sample_hop|k_hop|k_compact|k_count" --csv --log-file gpurun_out/ncu_sampler_part3.csv python tools/sampler_bench.py --config papers --reps 0 --paths part > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_part_tile --launch-skip 11 --launch-count 1 -o gpurun_out/prof_part_tile1 -f python tools/sampler_bench.py --config papers --reps 0 --paths part > /dev/null 2>&1
