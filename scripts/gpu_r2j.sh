#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/sync_probe.py 100 > gpurun_out/sync_probe.log 2>&1; echo probe=$?; cat gpurun_out/sync_probe.log
timeout 600 python -m pytest -q -x tests/test_gpu_frame_api.py > gpurun_out/pytest_api.log 2>&1; echo api=$?; tail -1 gpurun_out/pytest_api.log
