#!/bin/bash
# GPU-box session: smoke, GPU tests, bench (+ tuning variants), ncu launch list + one full capture.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [quick]
mkdir -p gpurun_out
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.log 2>&1; echo bench=$?
for v in paper_1911_06001_b200/lib_v*; do
  [ -d "$v" ] || continue
  VOXANIM_LIB_DIR=$PWD/$v timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_$(basename $v).log 2>&1
done
[ "$1" = quick ] && exit 0
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-extras --headstart-us 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frame_kernel -s 2 -c 1 -o gpurun_out/prof_frame $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
