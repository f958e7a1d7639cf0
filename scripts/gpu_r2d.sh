#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_frame_api.py > gpurun_out/pytest_parity.log 2>&1; echo parity=$?; tail -3 gpurun_out/pytest_parity.log
timeout 600 python scripts/debug_bugs.py > gpurun_out/debug_bugs_base.log 2>&1; echo dbg=$?; grep "==" gpurun_out/debug_bugs_base.log
timeout 900 python scripts/fp32_evidence.py gpurun_out/fp32_evidence.json > gpurun_out/fp32_evidence.log 2>&1; echo evidence=$?
