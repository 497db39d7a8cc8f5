set -x
timeout 300 python tools/debug_nonconvex.py > gpurun_out/r2d_nonconvex.log 2>&1
timeout 300 python tools/chol_trace.py C3 gpurun_out/trace_C3.npz > gpurun_out/r2d_trace_c3.log 2>&1
timeout 600 python tools/chol_trace.py C4 gpurun_out/trace_C4.npz > gpurun_out/r2d_trace_c4.log 2>&1
timeout 300 python tools/timeline.py C3 > gpurun_out/r2d_timeline_c3.log 2>&1
timeout 900 python bench.py --workload C4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench_c4.log 2>&1
timeout 900 python bench.py --workload C5 --batch 256 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2d_c5_256.log 2>&1
