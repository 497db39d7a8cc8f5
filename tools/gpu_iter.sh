# quick GPU iteration: chol + parity tests, C3 trace, short bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python tools/chol_trace.py C3 gpurun_out/trace_C3.npz > gpurun_out/trace.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
