# final tree: default bench line (C3 + C4 sub-record, e2e, CPU baseline), reference arm, smoke
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02final_smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/r02final_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/r02final_bench_ref.log 2>&1
ls gpurun_out/r02final*
