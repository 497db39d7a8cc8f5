timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2ao_pytest.log 2>&1
tail -n 2 gpurun_out/r2ao_pytest.log
timeout 300 python tools/timeline.py C3 > gpurun_out/r2ao_timeline.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-large > gpurun_out/r2ao_bench.log 2>&1
