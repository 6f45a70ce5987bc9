DGNN_ASM_TRACE=1 timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_t3.json 2> gpurun_out/r2_bench_t3.err
grep "asm-trace" gpurun_out/r2_bench_t3.err | grep -v "^\[asm-trace\] [0-9]:" 
