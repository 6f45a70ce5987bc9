timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/r2_gputests_full.log; cat gpurun_out/r2_gputests_full.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_final1.json 2> gpurun_out/r2_bench_final1.err; tail -2 gpurun_out/r2_bench_final1.err
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
