#!/bin/bash
# A/B of bench extras (C2/C3 1080p with and without the hit buffer, C4 FP64, crowd): in-tree lib vs lib_v*.
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for r in 0 1; do for v in paper_1911_06001_b200/lib paper_1911_06001_b200/lib_v*; do
  n=$(basename $v)
  VOXANIM_LIB_DIR=$PWD/$v timeout 600 $B > gpurun_out/abx_${n}_$r.log 2>&1
  python - "$n" gpurun_out/abx_${n}_$r.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1]); e = d["extras"]
print(sys.argv[1], {k: e[k]["ms_per_frame"] for k in ("c2_animated_1080p", "c3_static_1080p", "c2_animated_opt_1080p", "c3_static_opt_1080p", "c4_fp64")}, e["crowd_4096_4k"]["kernel_ms_per_frame"])
PY
done; done
