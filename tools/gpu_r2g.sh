# round-2 checkpoint: default bench line (C3 + C4 sub-record), reference arm,
# C3 launch list of one timed step
set -x
timeout 1500 python bench.py > gpurun_out/r02g_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r02g_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02g_launches_C3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large > /dev/null 2>&1
tail -c 3000 gpurun_out/r02g_bench.log
