# cluster size and stream-overlap switches at C4 / C3 after the top-share change
set -x
GN_TOP_CLUSTER=8 timeout 600 python bench.py --workload C4 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/knob_C4_cluster8.log 2>&1
GN_NO_OVERLAP=1 timeout 600 python bench.py --workload C4 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/knob_C4_nooverlap.log 2>&1
GN_NO_TOP_OVERLAP=1 timeout 600 python bench.py --workload C4 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/knob_C4_notopoverlap.log 2>&1
GN_TOP_CLUSTER=8 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-large > gpurun_out/knob_C3_cluster8.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-large > gpurun_out/knob_C3_default.log 2>&1
ls gpurun_out/knob*
