set -x
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2f_pytest_gpu.log 2>&1
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r2f_bench.log 2>&1
tail -n 3 gpurun_out/r2f_pytest_gpu.log
