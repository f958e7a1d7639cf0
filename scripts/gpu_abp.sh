#!/bin/bash
# A/B: C4 value, crowd kernel time and the partition shares (bench extras) of the in-tree lib and lib_v*.
mkdir -p gpurun_out
B="python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e"
for v in paper_1911_06001_b200/lib paper_1911_06001_b200/lib_v*; do
  n=$(basename $v)
  VOXANIM_LIB_DIR=$PWD/$v timeout 600 $B > gpurun_out/abp_${n}.log 2>&1
  python - "$n" gpurun_out/abp_${n}.log <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1]); e = d["extras"]; ps = e["partition_shares"]
print(sys.argv[1], "value", d["value"], "ms", d["ms_per_step"], "crowd", e["crowd_4096_4k"]["kernel_ms_per_frame"],
      "n1", ps["n1_ms"], {k: (ps[k]["max_ms"], ps[k]["compute_efficiency"]) for k in ("n2", "n4", "n8")})
PY
done
