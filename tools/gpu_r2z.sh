# prep kernels with register accumulators: parity suite, bench (C3 + C4)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02z_pytest.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02z_bench.log 2>&1
ls -la gpurun_out/r02z*
