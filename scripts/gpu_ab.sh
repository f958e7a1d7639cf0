#!/bin/bash
# A/B timing on the GPU box: the in-tree lib, every lib_v* variant, the in-tree lib again.
mkdir -p gpurun_out
B="python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-extras"
timeout 300 $B > gpurun_out/ab_base0.log 2>&1
for v in paper_1911_06001_b200/lib_v*; do
  [ -d "$v" ] || continue
  VOXANIM_LIB_DIR=$PWD/$v timeout 300 $B > gpurun_out/ab_$(basename $v).log 2>&1
done
timeout 300 $B > gpurun_out/ab_base1.log 2>&1
python scripts/show_bench.py gpurun_out/ab_*.log
# parity of each variant (FP32/FP64 parity suite); VARIANT_TESTS overrides the selection
for v in paper_1911_06001_b200/lib paper_1911_06001_b200/lib_v*; do
  [ -d "$v" ] || continue
  VOXANIM_LIB_DIR=$PWD/$v timeout 600 python -m pytest -q -x -m gpu ${VARIANT_TESTS:-tests/test_gpu_parity.py tests/test_gpu_fuzz.py} > gpurun_out/ab_pytest_$(basename $v).log 2>&1; echo "$v pytest=$? $(tail -1 gpurun_out/ab_pytest_$(basename $v).log)"
done
