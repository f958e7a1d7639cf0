"""Debug helper (not collected by pytest): print FP32-vs-oracle mismatch breakdowns on the GPU box."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1911_06001_b200 as vx  # noqa: E402
from oracle import ref  # noqa: E402


def report(name, s, o, culling=True, sorting=True, limit=6, classes=(2, 3)):
    o_aov, _ = o.dump(culling, sorting)
    _, aov, _ = s.render(culling, sorting, precision=vx.VXA_FP32, aov=True)
    cls = o.classify(o_aov, aov, 1e-6)
    print(f"== {name}: hits {(o_aov['object_id']>=0).sum()} match {(cls==0).sum()} tie {(cls==1).sum()} "
          f"bug {(cls==2).sum()} t_out {(cls==3).sum()}")
    for c in classes:
        ys, xs = np.nonzero(cls == c)
        print("  class", c, "pixels", list(zip(xs.tolist(), ys.tolist()))[:40])
        for y, x in list(zip(ys, xs))[:limit]:
            print(o.explain(int(x), int(y), o_aov[y, x], aov[y, x]))


def pair(cfg, models, seed=0, w=0, h=0):
    rmodels = [ref.RefModel.from_bytes(m.serialize()) for m in models]
    s = vx.Scene(cfg, models, seed, w, h)
    o = ref.RefScene(cfg, rmodels, seed, s.width, s.height)
    return s, o


if __name__ == "__main__":
    s, o = pair(vx.config.AXIS_ALIGNED, [vx.Model.procedural(6, shell=False), vx.Model.random(9, 4, 0.3)])
    report("axis aligned", s, o)
