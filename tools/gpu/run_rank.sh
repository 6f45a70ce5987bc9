timeout 900 python -m pytest tests/test_gpu_sampler_paths.py tests/test_gpu_blocks.py -m gpu -x -q 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/sampler_bench.py --config papers --reps 3 --paths part,part-sort,table --out gpurun_out/sampler_papers_rank.json 2> gpurun_out/sampler_papers_rank.err | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_rank.json 2> gpurun_out/r2_bench_rank.err; tail -1 gpurun_out/r2_bench_rank.json | head -c 600
