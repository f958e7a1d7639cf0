import ctypes as C, time, os
import paper_1911_06001_b200 as vx
lib=vx.vxa(); ctx=vx.context()
for depth in (8,10):
    words, gd = vx.grid_primitive("sphere", depth)
    lib.vxa_host_register(ctx, words.ctypes.data, words.nbytes)
    for r in range(3):
        h=C.c_uint32()
        t0=time.perf_counter()
        assert lib.vxa_build_model(ctx, words.ctypes.data, gd, 0, 0, C.byref(h), None, None)==0
        t1=time.perf_counter()
        lib.vxa_release_model(ctx, h.value)
        print(depth, r, "build %.2f ms release %.2f ms"%((t1-t0)*1e3,(time.perf_counter()-t1)*1e3), flush=True)
