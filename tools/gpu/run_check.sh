set -x
nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_gputests.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_20x5.json 2> gpurun_out/r2_bench_20x5.err
tail -3 gpurun_out/r2_bench_20x5.err
timeout 900 python bench.py --gpus 1 --steps 40 --warmup 5 > gpurun_out/r2_bench_40x5.json 2> gpurun_out/r2_bench_40x5.err
tail -3 gpurun_out/r2_bench_40x5.err
cat gpurun_out/r2_gputests.log
