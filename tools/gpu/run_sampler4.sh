timeout 900 python -m pytest tests/test_gpu_sampler_paths.py tests/test_gpu_blocks.py -m gpu -x -q 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/sampler_bench.py --config papers --reps 3 --out gpurun_out/sampler_papers4.json 2> gpurun_out/sampler_papers4.err | tail -1
DGNN_SAMPLE_HOP=warp DGNN_SAMPLE_COUNT=group timeout 600 python tools/sampler_bench.py --config papers --reps 2 --paths part 2>/dev/null | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_s4.json 2> gpurun_out/r2_bench_s4.err; tail -1 gpurun_out/r2_bench_s4.err
