timeout 900 python -m pytest tests/test_gpu_bench_runner.py tests/test_gpu_bench_contract.py -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_async.json 2> gpurun_out/r2_bench_async.err; tail -1 gpurun_out/r2_bench_async.err
DGNN_ASYNC_ASM=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_sync.json 2> gpurun_out/r2_bench_sync.err; tail -1 gpurun_out/r2_bench_sync.err
