"""Synchronous render_frame at C4 (the drop-in call, RGB8 into page-locked host
memory): wall time per call for the direct readback (the frame kernel stores
each finished super-tile's rows into the mapped host image) and for several
readback band counts (0 = one copy after the kernel), next to the frame
kernels' event time."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_06001_b200 as vx  # noqa: E402
from paper_1911_06001_b200 import _abi  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
lib, ctx = vx.vxa(), vx.context()
sc = vx.Scene(vx.config.C4, [vx.Model.procedural(11, shell=True)])
W, H = sc.width, sc.height
buf = np.empty((H, W, 3), np.uint8)
lib.vxa_host_register(ctx, buf.ctypes.data, buf.nbytes)
# (readback, option): direct with its super-tile order, or bands with one / two copy streams
CASES = [("direct", "screen"), ("direct", "banded"), ("direct", "lpt"), ("0", "2"), ("16", "2"), ("16", "1")]
for bands, opt in CASES:
    os.environ["VOXANIM_DIRECT_READBACK"] = "1" if bands == "direct" else "0"
    if bands == "direct":
        os.environ["VOXANIM_DIRECT_ORDER"] = opt
    else:
        os.environ["VOXANIM_READBACK_STREAMS"] = opt
    if bands in ("0", "direct"):
        os.environ["VOXANIM_BANDED_READBACK"] = "0"
    else:
        os.environ.pop("VOXANIM_BANDED_READBACK", None)
        os.environ["VOXANIM_READBACK_BANDS"] = bands
    for k in range(5):
        sc.evaluate(k / 30.0)
        sc.render(precision=vx.VXA_FP32, rgb=buf)
    host, gpu = [], []
    t0 = time.perf_counter()
    for k in range(steps):
        sc.evaluate(k / 30.0)
        a = time.perf_counter()
        st = sc.render(precision=vx.VXA_FP32, rgb=buf)[2]
        host.append(time.perf_counter() - a)
        gpu.append(st["gpu_ms"])
    el = (time.perf_counter() - t0) / steps
    print(f"readback {bands:>6} {opt:>6}: {el * 1e3:.3f} ms/step ({W * H / el / 1e6:.0f} Mrays/s), render call median "
          f"{np.median(host) * 1e3:.3f} ms, kernels (events) median {np.median(gpu):.3f} ms", flush=True)
