"""Renders a few frames of the CROWD configuration (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1911_06001_b200 as vx

count = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4
sc = vx.Scene(vx.config.CROWD, [vx.Model.procedural(8, shell=True)], count)
lib, vxl, ctx = vx.vxa(), vx.voxanim(), vx.context()
for k in range(frames):
    assert vxl.vxn_scene_submit(sc._h, k / 30.0, vx.VXA_FP32, 0, 1, 0) == 0
lib.vxa_synchronize(ctx)
print("ok")
