#!/bin/bash
# Quick A/B timing on the GPU box: the in-tree lib (compact + wide node words) plus every lib_v* variant build.
mkdir -p gpurun_out
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-extras > gpurun_out/bench.log 2>&1; echo bench=$?
VOXANIM_NODE_WORDS=wide timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-extras --no-e2e > gpurun_out/bench_wide.log 2>&1
for v in paper_1911_06001_b200/lib_v*; do
  [ -d "$v" ] || continue
  VOXANIM_LIB_DIR=$PWD/$v timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-extras > gpurun_out/bench_$(basename $v).log 2>&1
done
