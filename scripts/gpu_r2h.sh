#!/bin/bash
# A/B of the lib_v* variants against the in-tree lib, the whole GPU suite, the full bench.
mkdir -p gpurun_out
B="python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-extras"
timeout 300 $B > gpurun_out/ab_base0.log 2>&1
for v in paper_1911_06001_b200/lib_v*; do
  [ -d "$v" ] || continue
  VOXANIM_LIB_DIR=$PWD/$v timeout 300 $B > gpurun_out/ab_$(basename $v).log 2>&1
done
timeout 300 $B > gpurun_out/ab_base1.log 2>&1
python scripts/show_bench.py gpurun_out/ab_*.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.log 2>&1; echo bench=$?
