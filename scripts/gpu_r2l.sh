#!/bin/bash
# A/B vs lib_v*, whole GPU suite, full bench, FP32 evidence, ncu launch list + full capture.
mkdir -p gpurun_out
B="python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-extras"
timeout 300 $B > gpurun_out/ab_base0.log 2>&1
for v in paper_1911_06001_b200/lib_v*; do
  [ -d "$v" ] || continue
  VOXANIM_LIB_DIR=$PWD/$v timeout 300 $B > gpurun_out/ab_$(basename $v).log 2>&1
done
timeout 300 $B > gpurun_out/ab_base1.log 2>&1
python scripts/show_bench.py gpurun_out/ab_*.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 900 python scripts/fp32_evidence.py gpurun_out/fp32_evidence.json > gpurun_out/fp32_evidence.log 2>&1; echo evidence=$?
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --headstart-us 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frame_kernel -s 2 -c 1 -o gpurun_out/prof_frame $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
