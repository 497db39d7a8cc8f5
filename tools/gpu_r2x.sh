# top fronts with 16-column panels: rank 0 computes only the next panel half of the strip: parity suite, bench, C3/C4 traces
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02x_pytest.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02x_bench.log 2>&1
timeout 600 python tools/chol_trace.py C3 gpurun_out/r02x_trace_C3.npz > gpurun_out/r02x_trace_C3.log 2>&1
timeout 900 python tools/chol_trace.py C4 gpurun_out/r02x_trace_C4.npz > gpurun_out/r02x_trace_C4.log 2>&1
ls -la gpurun_out/r02x*
