# backward small sweep: two <=16-row fronts in flight per warp (tile halves)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/half_pytest.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/half_bench.log 2>&1
timeout 600 python tools/chol_trace.py C3 gpurun_out/half_trace_C3.npz > gpurun_out/half_trace_C3.log 2>&1
timeout 900 python tools/chol_trace.py C4 gpurun_out/half_trace_C4.npz > gpurun_out/half_trace_C4.log 2>&1
ls gpurun_out/half*
