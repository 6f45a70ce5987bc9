set -x
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_part|k_seed_sort|scan_kernel|k_sample_hop|k_hop|k_compact|k_count" --csv --log-file gpurun_out/ncu_sampler_part.csv python tools/sampler_bench.py --config papers --reps 0 --paths part > /dev/null 2> gpurun_out/ncu_sampler_part.err
tail -3 gpurun_out/ncu_sampler_part.err
