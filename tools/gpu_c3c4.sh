timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --workload C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4.log 2>&1
