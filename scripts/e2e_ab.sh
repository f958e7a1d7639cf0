#!/bin/bash
# e2e A/B on the GPU box: scripts/e2e_probe.py (streamed readback vs submission alone) for the
# in-tree lib and every lib_v* variant, then the bench's device-timed step for each.
mkdir -p gpurun_out
for v in paper_1911_06001_b200/lib paper_1911_06001_b200/lib_v* paper_1911_06001_b200/lib; do
  [ -d "$v" ] || continue
  echo "== $v"; VOXANIM_LIB_DIR=$PWD/$v PYTHONPATH=. timeout 300 python scripts/e2e_probe.py 300
done
bash scripts/gpu_ab.sh
