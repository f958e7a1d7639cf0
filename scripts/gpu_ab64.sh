#!/bin/bash
# FP64 parity kernel A/B: C4 bench at FP64, in-tree lib vs lib_v*; then the FP64 parity tests of the in-tree lib.
mkdir -p gpurun_out
B="python bench.py --precision fp64 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e --no-extras"
for r in 0 1; do for v in paper_1911_06001_b200/lib paper_1911_06001_b200/lib_v*; do
  VOXANIM_LIB_DIR=$PWD/$v timeout 300 $B > gpurun_out/ab64_$(basename $v)_$r.log 2>&1
done; done
python scripts/show_bench.py gpurun_out/ab64_*.log
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_traversal.py tests/test_reference_suites.py > gpurun_out/ab64_pytest.log 2>&1; echo "pytest=$? $(tail -1 gpurun_out/ab64_pytest.log)"
