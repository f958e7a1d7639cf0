#!/bin/bash
# Round-2 first GPU pass: new tests first, then the whole GPU suite, then the bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python -m pytest -x -q tests/test_gpu_frame_sync.py tests/test_gpu_multirank_bench.py tests/test_gpu_builder.py > gpurun_out/pytest_new.log 2>&1; echo new=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -c 600 gpurun_out/bench.log
