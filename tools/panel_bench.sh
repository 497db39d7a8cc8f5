#!/bin/bash
# build + run the panel microbenchmark (GPU box)
set -e
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Iinclude -Ipaper_2307_16830_b200/csrc \
  tools/panel_bench.cu -o /tmp/panel_bench -Lpaper_2307_16830_b200/_lib -lgridopf -Xlinker -rpath=$(pwd)/paper_2307_16830_b200/_lib
for a in "$@"; do timeout 30 stdbuf -o0 /tmp/panel_bench $a; echo "rc=$?"; done
