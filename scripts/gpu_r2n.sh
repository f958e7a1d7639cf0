#!/bin/bash
mkdir -p gpurun_out
bash scripts/gpu_r2k.sh
SEEDS=6000 MANY=400 HBO=400 bash scripts/gpu_soak.sh
