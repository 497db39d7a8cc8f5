timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload C5 --batch 32 --steps 2 --warmup 1 > gpurun_out/bench_c5.log 2>&1
timeout 900 python bench.py --workload C4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1
tail -c 1500 gpurun_out/bench_c4.log
