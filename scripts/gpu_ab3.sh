#!/bin/bash
# A/B under a time limit per run (variants that may hang): C4 bench + crowd + parity per variant.
mkdir -p gpurun_out
B="python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-extras"
for v in paper_1911_06001_b200/lib paper_1911_06001_b200/lib_v*; do
  n=$(basename $v)
  VOXANIM_LIB_DIR=$PWD/$v timeout 120 $B > gpurun_out/ab_${n}.log 2>&1; echo "$n bench=$?"
  echo "$n crowd $(VOXANIM_LIB_DIR=$PWD/$v timeout 120 python scripts/crowd_time.py 2>&1 | tail -1)"
done
python scripts/show_bench.py gpurun_out/ab_*.log
for v in paper_1911_06001_b200/lib_v*; do
  VOXANIM_LIB_DIR=$PWD/$v timeout 600 python -m pytest -q -x -m gpu ${VARIANT_TESTS:-tests/test_gpu_parity.py} > gpurun_out/ab_pytest_$(basename $v).log 2>&1; echo "$v pytest=$? $(tail -1 gpurun_out/ab_pytest_$(basename $v).log)"
done
