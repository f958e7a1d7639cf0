#!/bin/bash
# A/B: C4 bench + crowd kernel time, in-tree lib vs lib_v* variants; then parity of the in-tree lib.
mkdir -p gpurun_out
B="python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-extras"
for r in 0 1; do
  for v in paper_1911_06001_b200/lib paper_1911_06001_b200/lib_v*; do
    [ -d "$v" ] || continue
    n=$(basename $v)
    VOXANIM_LIB_DIR=$PWD/$v timeout 300 $B > gpurun_out/ab_${n}_$r.log 2>&1
    echo "$n crowd $(VOXANIM_LIB_DIR=$PWD/$v timeout 300 python scripts/crowd_time.py 2>&1 | tail -1)"
  done
done
python scripts/show_bench.py gpurun_out/ab_*.log
timeout 900 python -m pytest -q -x -m gpu ${VARIANT_TESTS:-tests/test_gpu_parity.py tests/test_gpu_fuzz.py} > gpurun_out/ab_pytest.log 2>&1; echo "pytest=$? $(tail -1 gpurun_out/ab_pytest.log)"
