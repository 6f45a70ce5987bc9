set -x
timeout 900 python -m pytest tests/test_gpu_sampler_paths.py tests/test_gpu_parity.py tests/test_gpu_blocks.py -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_sampler_tests.log
cat gpurun_out/r2_sampler_tests.log
timeout 600 python tools/sampler_bench.py --config papers --reps 3 --out gpurun_out/sampler_papers.json 2> gpurun_out/sampler_papers.err
tail -5 gpurun_out/sampler_papers.err
timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_bench_part.json 2> gpurun_out/r2_bench_part.err
tail -2 gpurun_out/r2_bench_part.err
