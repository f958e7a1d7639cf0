#!/bin/bash
# C4 bench (no readback) and the synchronous readback probe: in-tree lib vs lib_v* variants.
mkdir -p gpurun_out
B="python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-extras"
for v in paper_1911_06001_b200/lib paper_1911_06001_b200/lib_v*; do
  n=$(basename $v)
  VOXANIM_LIB_DIR=$PWD/$v timeout 300 $B > gpurun_out/ab_${n}.log 2>&1
  echo "== $n"; VOXANIM_LIB_DIR=$PWD/$v timeout 300 python scripts/sync_probe.py 100 2>&1
done
python scripts/show_bench.py gpurun_out/ab_*.log
timeout 600 python -m pytest -q -x tests/test_gpu_frame_api.py > gpurun_out/pytest_api.log 2>&1; echo api=$?; tail -1 gpurun_out/pytest_api.log
