# top-front cluster kernel beside the large-front kernel at C4 (forced) vs serial
set -x
GN_FORCE_TOP_OVERLAP=1 timeout 600 python bench.py --workload C4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/tov_C4_forced.log 2>&1
timeout 600 python bench.py --workload C4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/tov_C4_default.log 2>&1
GN_FORCE_TOP_OVERLAP=1 timeout 600 python bench.py --workload C4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/tov_C4_forced2.log 2>&1
ls gpurun_out/tov*
