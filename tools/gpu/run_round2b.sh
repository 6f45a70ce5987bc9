timeout 1200 python -m pytest tests/test_gpu_host_order.py tests/test_gpu_sharded_features.py tests/test_gpu_graph_chunk.py tests/test_gpu_bench_contract.py tests/test_gpu_diskcache.py -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_ho.json 2> gpurun_out/r2_bench_ho.err; tail -2 gpurun_out/r2_bench_ho.err
DGNN_HOST_ORDER=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_noho.json 2> gpurun_out/r2_bench_noho.err; tail -1 gpurun_out/r2_bench_noho.err
