timeout 900 python -m pytest tests/test_gpu_chol.py tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2ah_pytest.log 2>&1
timeout 300 python tools/chol_trace.py C3 gpurun_out/trace_C3_ni_old.npz > gpurun_out/r2ah_trace.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2ah_bench.log 2>&1
