"""Where does the e2e step time go? Streams C4 frames like bench.py's e2e and
reports the wall time per step next to the frame kernels' own event time."""
import ctypes as C
import sys
import time

import numpy as np

import paper_1911_06001_b200 as vx
from paper_1911_06001_b200 import _abi

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
lib, vxl, ctx = vx.vxa(), vx.voxanim(), vx.context()
sc = vx.Scene(vx.config.C4, [vx.Model.procedural(11, shell=True)])
W, H = sc.width, sc.height
bufs = [np.empty((H, W, 3), np.uint8) for _ in range(3)]
for b in bufs:
    lib.vxa_host_register(ctx, b.ctypes.data, b.nbytes)
t = C.c_uint64()
for mode in ("stream", "stream3", "submit_only"):
    tickets = []
    for k in range(5):
        vxl.vxn_scene_stream(sc._h, k / 30.0, vx.VXA_FP32, bufs[k % 2].ctypes.data, C.byref(t))
    lib.vxa_synchronize(ctx)
    lib.vxa_stats_reset(ctx)
    t0 = time.perf_counter()
    t_sub = t_wait = 0.0  # host time inside the submission call / blocked in the wait
    for k in range(steps):
        if mode.startswith("stream"):
            depth = 3 if mode == "stream3" else 2  # host images in flight
            a = time.perf_counter()
            vxl.vxn_scene_stream(sc._h, k / 30.0, vx.VXA_FP32, bufs[k % depth].ctypes.data, C.byref(t))
            b = time.perf_counter()
            tickets.append(t.value)
            if len(tickets) >= depth:
                lib.vxa_wait_readback(ctx, tickets[-depth])
            t_sub += b - a
            t_wait += time.perf_counter() - b
        else:
            vxl.vxn_scene_submit(sc._h, k / 30.0, vx.VXA_FP32, 0, 1, 0)
    if mode.startswith("stream"):
        lib.vxa_wait_readback(ctx, tickets[-1])
    lib.vxa_synchronize(ctx)
    el = (time.perf_counter() - t0) * 1e3 / steps
    st = _abi.vxa_stats()
    lib.vxa_stats_read(ctx, C.byref(st))
    print(f"{mode:12s} wall {el:.4f} ms/step   frame kernels {st.gpu_ms / st.frames:.4f} ms/frame ({st.frames} frames)"
          + (f"   host: submit {t_sub * 1e3 / steps:.4f} ms, wait {t_wait * 1e3 / steps:.4f} ms per step"
             if mode.startswith("stream") else ""))

# D2H bandwidth of one RGB8 frame into page-locked host memory (torch, for reference)
import torch

src = torch.empty(W * H * 3, dtype=torch.uint8, device="cuda")
dst = torch.empty(W * H * 3, dtype=torch.uint8, pin_memory=True)
for _ in range(3):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
el = (time.perf_counter() - t0) / 20
print(f"D2H {W * H * 3 / 1e6:.1f} MB: {el * 1e3:.3f} ms ({W * H * 3 / el / 1e9:.1f} GB/s)")
