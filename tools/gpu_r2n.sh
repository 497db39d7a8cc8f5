# round-2 re-entry: GPU suite, default bench (C3 + C4 sub-record), reference
# arm, C3 launch list, C5 batch
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02n_pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/r02n_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r02n_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02n_launches_C3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large > /dev/null 2>&1
timeout 1200 python bench.py --workload C5 --batch 256 --steps 3 --warmup 3 > gpurun_out/r02n_bench_C5.log 2>&1
ls -la gpurun_out/r02n*
