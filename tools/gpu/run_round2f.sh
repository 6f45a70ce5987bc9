timeout 900 python -m pytest tests/test_gpu_sampler_paths.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
DGNN_ASM_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_g.json 2> gpurun_out/r2_bench_g.err; tail -1 gpurun_out/r2_bench_g.err
DGNN_ASM_PRIORITY=-1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_gp.json 2> gpurun_out/r2_bench_gp.err; tail -1 gpurun_out/r2_bench_gp.err
