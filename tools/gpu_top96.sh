# kTopFronts 24 -> 96: GPU suite, default bench (C3 + C4), C4 at 64 / 128 top fronts
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/top96_pytest.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/top96_bench.log 2>&1
for TF in 64 128; do
  GN_TOP_FRONTS=$TF timeout 600 python bench.py --workload C4 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/top_sweep_C4_$TF.log 2>&1
done
timeout 600 python tools/chol_trace.py C4 gpurun_out/top96_trace_C4.npz > gpurun_out/top96_trace_C4.log 2>&1
ls gpurun_out/top*
