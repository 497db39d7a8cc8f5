# round-2 profiles: launch lists (time + DRAM bytes) and --set full captures
# of the hot kernels at C2 and C4 (tools/kernels_once.py), plus a C3 launch list
set -x
for WL in C2 C4; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"mf_|gn_ad|ad_gather|ad_objective|assemble_kernel|d_rows" \
  --log-file gpurun_out/r02c_launches_$WL.csv python tools/kernels_once.py $WL 2 > gpurun_out/r02c_launches_$WL.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"mf_factor|mf_forward|mf_backward|gn_ad_patterns|assemble_kernel" -c 12 \
  -o gpurun_out/r02c_full_$WL -f python tools/kernels_once.py $WL 1 > gpurun_out/r02c_full_$WL.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02c_launches_C3_step.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-large > /dev/null 2>&1
ls -la gpurun_out/r02c*
