timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2am_pytest.log 2>&1
tail -n 2 gpurun_out/r2am_pytest.log
timeout 300 python tools/chol_trace.py C4 gpurun_out/trace_C4_split.npz > /dev/null 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2am_bench.log 2>&1
