#!/bin/bash
for b in 16 8; do echo "bands $b"; BANDS=$b bash scripts/band_trace.sh; done
timeout 300 python scripts/sync_probe.py 100 2>&1 | tail -5
timeout 600 python -m pytest -q -x tests/test_gpu_frame_api.py 2>&1 | tail -1
