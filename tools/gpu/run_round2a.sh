timeout 900 python -m pytest tests/test_gpu_graph_chunk.py tests/test_gpu_bench_contract.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_part2.json 2> gpurun_out/r2_bench_part2.err; tail -1 gpurun_out/r2_bench_part2.err
DGNN_SAMPLE_DEDUP=table timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_table2.json 2> gpurun_out/r2_bench_table2.err; tail -1 gpurun_out/r2_bench_table2.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --stage file > gpurun_out/r2_bench_file.json 2> gpurun_out/r2_bench_file.err; tail -3 gpurun_out/r2_bench_file.err
df -h /tmp . | tail -2; nproc; free -g | head -2
