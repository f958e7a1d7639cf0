#!/bin/bash
# Round-2 evidence pass: GPU suite, smoke, full bench, FP32 evidence, sync probe,
# ncu launch list + one full capture of the C4 frame kernel and of the 4096-instance crowd.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 900 python scripts/fp32_evidence.py gpurun_out/fp32_evidence.json > gpurun_out/fp32_evidence.log 2>&1; echo evidence=$?
timeout 300 python scripts/sync_probe.py 100 > gpurun_out/sync_probe.log 2>&1; echo probe=$?
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --headstart-us 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frame_kernel -s 2 -c 1 -o gpurun_out/prof_frame $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 300 python scripts/crowd_frames.py 4096 4 > gpurun_out/crowd_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frame_kernel -s 2 -c 1 -o gpurun_out/prof_crowd python scripts/crowd_frames.py 4096 4 > gpurun_out/ncu_crowd.log 2>&1; echo ncu3=$?
