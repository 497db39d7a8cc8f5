# trailing update in 32x16 halves, A22 loads overlapping the DMMAs: parity suite, bench, C3/C4 traces
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02v_pytest.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02v_bench.log 2>&1
timeout 600 python tools/chol_trace.py C3 gpurun_out/r02v_trace_C3.npz > gpurun_out/r02v_trace_C3.log 2>&1
timeout 900 python tools/chol_trace.py C4 gpurun_out/r02v_trace_C4.npz > gpurun_out/r02v_trace_C4.log 2>&1
ls -la gpurun_out/r02v*
