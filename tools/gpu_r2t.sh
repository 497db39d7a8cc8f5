# backward small-front sweep with counter-target barrier: parity suite, bench, C3 trace
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02t_pytest.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02t_bench.log 2>&1
timeout 600 python tools/chol_trace.py C3 gpurun_out/r02t_trace_C3.npz > gpurun_out/r02t_trace_C3.log 2>&1
ls -la gpurun_out/r02t*
