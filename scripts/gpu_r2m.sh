#!/bin/bash
mkdir -p gpurun_out
bash scripts/gpu_r2k.sh
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --headstart-us 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 300 python scripts/crowd_frames.py 4096 4 > gpurun_out/crowd_plain.log 2>&1; echo crowd=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frame_kernel -s 2 -c 1 -o gpurun_out/prof_crowd python scripts/crowd_frames.py 4096 4 > gpurun_out/ncu_crowd.log 2>&1; echo ncu3=$?
