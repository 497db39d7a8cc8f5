# sweep of the cluster-kernel share (GN_TOP_FRONTS) at C4 and C3
set -x
for TF in 24 48 96 192; do
  GN_TOP_FRONTS=$TF timeout 600 python bench.py --workload C4 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/top_sweep_C4_$TF.log 2>&1
done
for TF in 24 48 96; do
  GN_TOP_FRONTS=$TF timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-large > gpurun_out/top_sweep_C3_$TF.log 2>&1
done
ls gpurun_out/top_sweep*
