set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > gpurun_out/r2c_pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2c_bench.log 2>&1
timeout 900 python bench.py --workload C5 --batch 64 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2c_c5_64.log 2>&1
tail -3 gpurun_out/r2c_*.log
