"""Renders a few C4 frames at a given precision (for ncu captures): python scripts/c4_frames.py fp64 4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1911_06001_b200 as vx  # noqa: E402

prec = vx.VXA_FP64 if (len(sys.argv) > 1 and sys.argv[1] == "fp64") else vx.VXA_FP32
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4
sc = vx.Scene(vx.config.C4, [vx.Model.procedural(11, shell=True)])
lib, vxl, ctx = vx.vxa(), vx.voxanim(), vx.context()
for k in range(frames):
    assert vxl.vxn_scene_submit(sc._h, k / 30.0, prec, 0, 1, 0) == 0
lib.vxa_synchronize(ctx)
print("ok")
