# per-front timelines of one refactorisation + solve at C3 and C4
set -x
timeout 600 python tools/chol_trace.py C3 gpurun_out/r02r_trace_C3.npz > gpurun_out/r02r_trace_C3.log 2>&1
timeout 900 python tools/chol_trace.py C4 gpurun_out/r02r_trace_C4.npz > gpurun_out/r02r_trace_C4.log 2>&1
ls -la gpurun_out/r02r*
