# round-2 final profiles: default bench (C3 + C4 sub-record), reference arm,
# C3 launch list of one timed step, ncu --set full of one C3
# refactorisation + solve (tools/kernels_once.py) and of C4's, C5 batch.
set -x
timeout 1500 python bench.py > gpurun_out/r02h_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r02h_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02h_launches_C3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large > /dev/null 2>&1
for WL in C3 C4; do
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"mf_factor|mf_forward|mf_backward|gn_ad_patterns|assemble_kernel" -c 12 \
  -o gpurun_out/r02h_full_$WL -f python tools/kernels_once.py $WL 1 > gpurun_out/r02h_full_$WL.log 2>&1
done
timeout 1200 python bench.py --workload C5 --batch 256 --steps 3 --warmup 3 > gpurun_out/r02h_bench_C5.log 2>&1
ls -la gpurun_out/r02h*
