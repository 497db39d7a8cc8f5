# round-2 closing measurement (final tree): GPU suite, smoke, default bench
# (C3 + C4 sub-record, e2e, CPU baseline), reference arm, C3 launch list,
# ncu --set full of the hot kernels at C3 and C4 (reports kept on the box
# under /tmp, only their summaries and the raw metric pages come back), C5
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02y_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02y_smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/r02y_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r02y_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02y_launches_C3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large > /dev/null 2>&1
mkdir -p /tmp/ncu
for WL in C3 C4; do
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"mf_factor|mf_forward|mf_backward|gn_ad_patterns|ad_gather|assemble_kernel" -c 14 \
  -o /tmp/ncu/r02y_full_$WL -f python tools/kernels_once.py $WL 1 > gpurun_out/r02y_full_$WL.log 2>&1
python tools/ncu_full_summary.py /tmp/ncu/r02y_full_$WL.ncu-rep > gpurun_out/r02y_full_$WL.txt 2>&1
ncu -i /tmp/ncu/r02y_full_$WL.ncu-rep --page raw --csv > gpurun_out/r02y_full_${WL}_raw.csv 2>/dev/null
done
timeout 1200 python bench.py --workload C5 --batch 256 --steps 3 --warmup 3 > gpurun_out/r02y_bench_C5.log 2>&1
ls -la gpurun_out/
du -sh gpurun_out
