#!/bin/bash
# build + run the single-tile trailing-update microbenchmark (GPU box)
set -e
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Iinclude -Ipaper_2307_16830_b200/csrc \
  tools/tile_probe.cu -o /tmp/tile_probe -Lpaper_2307_16830_b200/_lib -lgridopf -Xlinker -rpath=$(pwd)/paper_2307_16830_b200/_lib
timeout 60 /tmp/tile_probe
