# sweep of the top-front minimum height (GN_TOP_MIN_ROWS) and count at C3 and C4
set -x
for TR in 48 64 80; do for TF in 96 192; do
  GN_TOP_MIN_ROWS=$TR GN_TOP_FRONTS=$TF timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-large > gpurun_out/toprows_C3_${TR}_${TF}.log 2>&1
done; done
for TR in 64 80 128; do
  GN_TOP_MIN_ROWS=$TR timeout 600 python bench.py --workload C4 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/toprows_C4_${TR}_96.log 2>&1
done
ls gpurun_out/toprows*
