# reduction grid 296 -> 1184 CTAs: parity suite + bench (C3 + C4 sub-record)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02p_pytest.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02p_bench.log 2>&1
ls -la gpurun_out/r02p*
