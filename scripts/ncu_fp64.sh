#!/bin/bash
mkdir -p gpurun_out
S="--section SourceCounters --section InstructionStats --section LaunchStats --section Occupancy --section SpeedOfLight --section WarpStateStats --section ComputeWorkloadAnalysis"
timeout 300 python scripts/c4_frames.py fp64 3 > gpurun_out/fp64_plain.log 2>&1 && \
timeout 900 ncu $S --clock-control none --import-source on -k regex:frame_kernel -s 2 -c 1 -o gpurun_out/src_fp64 python scripts/c4_frames.py fp64 3 > gpurun_out/ncu_fp64.log 2>&1; echo fp64=$?
