# AD contributions stored in gather order: parity suite, bench (C3 + C4), ncu
# of the AD kernels at C4 (compare r02o_full_ad_C4)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02q_pytest.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02q_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"gn_ad_patterns|ad_gather" -c 6 \
  -o gpurun_out/r02q_full_ad_C4 -f python tools/kernels_once.py C4 1 > gpurun_out/r02q_full_ad_C4.log 2>&1
ls -la gpurun_out/r02q*
