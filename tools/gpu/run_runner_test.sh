timeout 1500 python -m pytest tests/test_gpu_papers_runner.py tests/test_gpu_bench_contract.py -m gpu -x -q 2>&1 | tail -15
