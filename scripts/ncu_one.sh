#!/bin/bash
# One ncu --set full capture of a kernel (regex $1) from a short bench run; $2: launches to skip.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${2:-2} -c 1 -o gpurun_out/prof_${3:-frame} $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
