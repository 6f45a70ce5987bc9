timeout 1500 python -m pytest tests/test_gpu_sampler_paths.py tests/test_gpu_host_order.py tests/test_gpu_bench_runner.py tests/test_gpu_graph_chunk.py -m gpu -x -q 2>&1 | tail -4
timeout 600 python tools/sampler_bench.py --config papers --reps 3 --paths part 2> /dev/null | tail -1
DGNN_ASM_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_wspan.json 2> gpurun_out/r2_bench_wspan.err; grep "asm-trace" gpurun_out/r2_bench_wspan.err | head -12; tail -1 gpurun_out/r2_bench_wspan.err
