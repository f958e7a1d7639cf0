#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-extras"
for r in 0 1; do for v in paper_1911_06001_b200/lib paper_1911_06001_b200/lib_v*; do
  VOXANIM_LIB_DIR=$PWD/$v timeout 300 $B > gpurun_out/ab_$(basename $v)_$r.log 2>&1
done; done
python scripts/show_bench.py gpurun_out/ab_*.log
for r in 0 1; do timeout 300 python scripts/sync_probe.py 100 > gpurun_out/sync_probe_$r.log 2>&1; echo probe=$?; cat gpurun_out/sync_probe_$r.log; done
timeout 600 python -m pytest -q -x tests/test_gpu_frame_api.py > gpurun_out/pytest_api.log 2>&1; echo api=$?; tail -1 gpurun_out/pytest_api.log
