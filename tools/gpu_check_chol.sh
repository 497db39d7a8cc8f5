set -x
timeout 900 python -m pytest tests/test_gpu_chol.py tests/test_gpu_parity.py tests/test_gpu_ipm.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
true
