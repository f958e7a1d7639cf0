#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-extras"
timeout 300 $B > gpurun_out/ab_base0.log 2>&1
for v in paper_1911_06001_b200/lib_v*; do
  [ -d "$v" ] || continue
  VOXANIM_LIB_DIR=$PWD/$v timeout 300 $B > gpurun_out/ab_$(basename $v).log 2>&1
done
timeout 300 $B > gpurun_out/ab_base1.log 2>&1
python scripts/show_bench.py gpurun_out/ab_*.log
for v in paper_1911_06001_b200/lib_v*; do
  [ -d "$v" ] || continue
  VOXANIM_LIB_DIR=$PWD/$v timeout 600 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_traversal.py tests/test_gpu_frame_api.py > gpurun_out/pytest_$(basename $v).log 2>&1; echo $v=$?; tail -1 gpurun_out/pytest_$(basename $v).log
done
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_frame_api.py > gpurun_out/pytest_base.log 2>&1; echo base=$?; tail -1 gpurun_out/pytest_base.log
