#!/bin/bash
# Soak run of the randomized parity sweeps (FP64 bit-exact, FP32 ties only) at widened sizes.
mkdir -p gpurun_out
VOXANIM_FUZZ_SEEDS=${SEEDS:-600} VOXANIM_FUZZ_SEEDS_MANY=${MANY:-80} VOXANIM_FUZZ_SEEDS_HBO=${HBO:-80} timeout 2400 \
  python -m pytest -q tests/test_gpu_fuzz.py -k "random_scene or many or hbo" > gpurun_out/soak.log 2>&1; echo soak=$?
tail -5 gpurun_out/soak.log
grep -E "^E |FAILED" gpurun_out/soak.log | head -20
