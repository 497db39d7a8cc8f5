timeout 1200 python -m pytest tests/test_batch.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2aq_pytest.log 2>&1
tail -n 2 gpurun_out/r2aq_pytest.log
timeout 600 python tools/timeline_c5.py 256 > gpurun_out/r2aq_c5.log 2>&1
timeout 900 python bench.py --workload C5 --batch 256 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2aq_c5_bench.log 2>&1
