"""Crowd (4096 animated instances, 3840x2160) kernel time per frame: bench.crowd_bench."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1911_06001_b200 as vx  # noqa: E402

prec = vx.VXA_FP32 if (len(sys.argv) < 2 or sys.argv[1] == "fp32") else vx.VXA_FP64
r = bench.crowd_bench(vx.vxa(), vx.context(), vx.voxanim(), prec, frames=30)
print(json.dumps({k: r[k] for k in ("kernel_ms_per_frame", "mrays_per_s_kernel")}))
