#!/bin/bash
# ncu source counters of the crowd frame kernel (4096 instances) and of the C4 frame kernel.
mkdir -p gpurun_out
S="--section SourceCounters --section InstructionStats --section LaunchStats --section Occupancy --section SpeedOfLight --section WarpStateStats --section MemoryWorkloadAnalysis"
timeout 300 python scripts/crowd_frames.py 4096 4 > gpurun_out/crowd_plain.log 2>&1 && \
timeout 900 ncu $S --clock-control none --import-source on -k regex:frame_kernel -s 2 -c 1 -o gpurun_out/src_crowd python scripts/crowd_frames.py 4096 4 > gpurun_out/ncu_crowd.log 2>&1; echo crowd=$?
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-extras --headstart-us 0"
timeout 900 ncu $S --clock-control none --import-source on -k regex:frame_kernel -s 2 -c 1 -o gpurun_out/src_c4 $CMD > gpurun_out/ncu_c4.log 2>&1; echo c4=$?
