# End-of-round capture: C3 bench (full line), reference arm, ncu launch list,
# ncu --set full of one refactorisation (small + large + top kernels), C4 and
# C5 bench lines.  Outputs under gpurun_out/.
set -x
timeout 1200 python bench.py > gpurun_out/bench_C3.log 2>&1
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_C3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_C3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mf_factor -c 3 -s 9 \
    -o gpurun_out/factor_full -f python tools/chol_once.py C3 > gpurun_out/ncu_factor_full.log 2>&1
timeout 1200 python bench.py --workload C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4.log 2>&1
timeout 1200 python bench.py --workload C5 --batch 32 --steps 3 --warmup 3 > gpurun_out/bench_C5.log 2>&1
true
