"""Where the screen partition bottoms out (GPU box): C4 rendered as rank r of N on
one GPU for fine partitions (N = 255: 8 super-tiles per rank; N = 2040: one
super-tile per rank, every third one sampled); prints the max / median / min
device time of a share (CUDA events, best of 3 frames, L2 not flushed)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_06001_b200 as vx  # noqa: E402
from paper_1911_06001_b200 import _abi  # noqa: E402

lib, ctx, vxl = vx.vxa(), vx.context(), vx.voxanim()
scene = vx.Scene(vx.config.C4, [vx.Model.procedural(11, shell=True)])


def share_ms(rank, world, frames=3):
    vxl.vxn_scene_submit(scene._h, 0.4, _abi.VXA_FP32, rank, world, 0)
    lib.vxa_synchronize(ctx)
    best = []
    for _ in range(frames):
        lib.vxa_stream_delay(ctx, 300)
        lib.vxa_timer_begin(ctx)
        vxl.vxn_scene_submit(scene._h, 0.4, _abi.VXA_FP32, rank, world, 0)
        ms = C.c_double()
        lib.vxa_timer_end(ctx, C.byref(ms))
        best.append(ms.value)
    return min(best)


for world in (255, 2040):
    t = np.array([share_ms(r, world) for r in (range(world) if world <= 255 else range(0, world, 3))])
    print(world, "max %.4f median %.4f min %.4f" % (t.max(), np.median(t), t.min()),
          "top5", np.round(np.sort(t)[-5:], 4), flush=True)
