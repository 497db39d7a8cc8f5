set -x
timeout 600 python tools/debug_nonconvex.py > gpurun_out/r2b_nonconvex.log 2>&1
timeout 1200 python -m pytest tests/test_batch.py -m gpu -q -x > gpurun_out/r2b_batch.log 2>&1
timeout 900 python bench.py --workload C5 --batch 64 --steps 2 --warmup 1 > gpurun_out/r2b_c5_64.log 2>&1
timeout 900 python bench.py --workload C5 --batch 256 --steps 2 --warmup 1 > gpurun_out/r2b_c5_256.log 2>&1
