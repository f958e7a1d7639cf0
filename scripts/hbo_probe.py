"""Per-frame cost of the reference bench modes on the acceptance bench scene:
call wall time (FrameStats.render_ms) vs the frame kernels' own time."""
import os
import sys
import tempfile

sys.path.insert(0, "tools")
import paper_1911_06001_b200 as vx
from acceptance_perf import build_fixture

with tempfile.TemporaryDirectory() as d:
    build_fixture(vx, d)
    for label, cull, hbo_on in (("no-opt", False, False), ("cull+sort", True, False), ("cull+sort+hbo", True, True),
                                ("hbo only", False, True)):
        sc = vx.Scene.load(os.path.join(d, "bench.json"), 640, 480)
        hbo = vx.HitBuffer(640, 480) if hbo_on else None
        sc.render(culling=cull, sorting=cull)
        ms, gms = [], []
        for k in range(60):
            sc.evaluate(k / 30.0)
            _, _, st = sc.render(culling=cull, sorting=cull, hbo=hbo)
            sc.mark_clean()
            ms.append(st["render_ms"])
            gms.append(st["gpu_ms"])
        print(f"{label:14s} render_ms {sum(ms)/60:.4f}  kernel_ms {sum(gms)/60:.4f}  first {ms[0]:.3f}")
