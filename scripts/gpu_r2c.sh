#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/debug_bugs.py > gpurun_out/debug_bugs_base.log 2>&1; echo dbg=$?
VOXANIM_LIB_DIR=$PWD/paper_1911_06001_b200/lib_vold timeout 600 python scripts/debug_bugs.py > gpurun_out/debug_bugs_old.log 2>&1; echo dbg_old=$?
B="python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-extras"
timeout 300 $B > gpurun_out/ab_base0.log 2>&1
for v in paper_1911_06001_b200/lib_v*; do
  [ -d "$v" ] || continue
  VOXANIM_LIB_DIR=$PWD/$v timeout 300 $B > gpurun_out/ab_$(basename $v).log 2>&1
done
timeout 300 $B > gpurun_out/ab_base1.log 2>&1
python scripts/show_bench.py gpurun_out/ab_*.log
