#!/bin/bash
# build + run the solve-block microbenchmark (GPU box); tools/tile_bench.cu
# belongs to the tile-DAG experiment (branch dag-experiment)
set -e
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Iinclude -Ipaper_2307_16830_b200/csrc \
  tools/fwd_bench.cu -o /tmp/fwd_bench -Lpaper_2307_16830_b200/_lib -lgridopf -Xlinker -rpath=$(pwd)/paper_2307_16830_b200/_lib
timeout 30 /tmp/fwd_bench
