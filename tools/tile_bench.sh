#!/bin/bash
# build + run the PANEL microbenchmark (GPU box)
set -e
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Iinclude -Ipaper_2307_16830_b200/csrc \
  tools/tile_bench.cu -o /tmp/tile_bench -Lpaper_2307_16830_b200/_lib -lgridopf -Xlinker -rpath=$(pwd)/paper_2307_16830_b200/_lib
for m in dd rand; do echo $m; timeout 60 /tmp/tile_bench $m; done
