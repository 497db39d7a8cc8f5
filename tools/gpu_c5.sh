timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
for c in 1 2 4 8; do timeout 900 python bench.py --workload C5 --batch 64 --steps 2 --warmup 1 --concurrency $c > gpurun_out/bench_c5_$c.log 2>&1; done
