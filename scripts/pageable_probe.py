"""Synchronous render_frame into pageable host memory at C4 (the drop-in `Image`
case): wall time per call, against the page-locked (registered) case."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_06001_b200 as vx  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
lib, ctx = vx.vxa(), vx.context()
sc = vx.Scene(vx.config.C4, [vx.Model.procedural(11, shell=True)])
W, H = sc.width, sc.height
pageable = np.empty((H, W, 3), np.uint8)
pageable[...] = 1  # touched: no first-touch faults inside the timed calls
pinned = np.empty((H, W, 3), np.uint8)
lib.vxa_host_register(ctx, pinned.ctypes.data, pinned.nbytes)
for name, buf in (("pageable", pageable), ("registered", pinned), ("fresh numpy per call", None)):
    for k in range(5):
        sc.evaluate(k / 30.0)
        sc.render(precision=vx.VXA_FP32, rgb=buf if buf is not None else True)
    t0 = time.perf_counter()
    for k in range(steps):
        sc.evaluate(k / 30.0)
        sc.render(precision=vx.VXA_FP32, rgb=buf if buf is not None else True)
    el = (time.perf_counter() - t0) / steps
    print(f"{name:>22}: {el * 1e3:.3f} ms per call ({W * H / el / 1e6:.0f} Mrays/s)", flush=True)

# the drop-in voxanim::render_frame (Image by value), through the staging path and
# (VOXANIM_IMAGE_STAGING=0) rendering straight into the fresh Image
vxl = vx.voxanim()
ms = C.c_double()
for staged, spares in (("1", "1"), ("1", "0"), ("0", "0")):
    os.environ["VOXANIM_IMAGE_STAGING"] = staged
    os.environ["VOXANIM_IMAGE_SPARES"] = spares
    sc2 = vx.Scene(vx.config.C4, [vx.Model.procedural(11, shell=True)])
    assert vxl.vxn_scene_render_image(sc2._h, 0.0, 5, C.byref(ms), None) == 0  # warm-up
    last = np.empty((H, W, 3), np.uint8)
    assert vxl.vxn_scene_render_image(sc2._h, 1.0, steps, C.byref(ms), last.ctypes.data) == 0
    sc3 = vx.Scene(vx.config.C4, [vx.Model.procedural(11, shell=True)])
    sc3.evaluate(1.0 + (steps - 1) / 30.0)
    same = (sc3.render(precision=vx.VXA_FP32)[0] == last).all()
    print(f"{'render_frame (Image)':>22} staging={staged} spares={spares}: {ms.value:.3f} ms per call "
          f"({W * H / ms.value / 1e3:.0f} Mrays/s), image equals render_frame_into: {same}", flush=True)
