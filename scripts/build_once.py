"""Builds the depth-10 dense sphere on the device a few times (for ncu launch lists)."""
import ctypes as C
import sys

import paper_1911_06001_b200 as vx

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 10
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lib, ctx = vx.vxa(), vx.context()
words, gd = vx.grid_primitive("sphere", depth)
for _ in range(reps):
    h = C.c_uint32()
    assert lib.vxa_build_model(ctx, words.ctypes.data, gd, 0, 0, C.byref(h), None, None) == 0
    lib.vxa_release_model(ctx, h.value)
print("ok")
