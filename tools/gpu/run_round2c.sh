timeout 900 python -m pytest tests/test_gpu_host_order.py tests/test_gpu_diskcache.py -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_ho2.json 2> gpurun_out/r2_bench_ho2.err; tail -1 gpurun_out/r2_bench_ho2.err
timeout 600 python tools/diskcache_bench.py --config papers --fractions 0.95 > gpurun_out/diskcache_papers_r2.json 2>/dev/null; tail -c 600 gpurun_out/diskcache_papers_r2.json
timeout 600 python tools/diskcache_bench.py --config products --fractions 0.95,0.8,0.7 > gpurun_out/diskcache_products_r2.json 2>/dev/null; tail -c 300 gpurun_out/diskcache_products_r2.json
timeout 1500 python -m pytest tests/test_gpu_papers_runner.py -m gpu -x -q 2>&1 | tail -4
