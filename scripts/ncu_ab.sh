#!/bin/bash
# ncu source-counter captures of the frame kernel: in-tree lib and every lib_v* variant.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-extras --headstart-us 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 || exit 1
timeout 600 ncu --section SourceCounters --section InstructionStats --section LaunchStats --section Occupancy --section SpeedOfLight --section WarpStateStats --clock-control none --import-source on -k regex:frame_kernel -s 2 -c 1 -o gpurun_out/src_base $CMD > gpurun_out/ncu_base.log 2>&1; echo base=$?
for v in paper_1911_06001_b200/lib_v*; do
  [ -d "$v" ] || continue
  VOXANIM_LIB_DIR=$PWD/$v timeout 600 ncu --section SourceCounters --section InstructionStats --section LaunchStats --section Occupancy --section SpeedOfLight --section WarpStateStats --clock-control none --import-source on -k regex:frame_kernel -s 2 -c 1 -o gpurun_out/src_$(basename $v) $CMD > gpurun_out/ncu_$(basename $v).log 2>&1; echo $v=$?
done
