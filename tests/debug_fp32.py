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
        for y, x in list(zip(ys, xs))[:limit]:
            print(o.explain(int(x), int(y), o_aov[y, x], aov[y, x]))
            print("   rel err", abs(o_aov[y, x]['t'] - aov[y, x]['t']) / max(1, abs(o_aov[y, x]['t'])))


def pair(cfg, models, seed=0, w=0, h=0):
    rmodels = [ref.RefModel.from_bytes(m.serialize()) for m in models]
    s = vx.Scene(cfg, models, seed, w, h)
    o = ref.RefScene(cfg, rmodels, seed, s.width, s.height)
    return s, o


if __name__ == "__main__":
    s, o = pair(2, [vx.Model.procedural(10, shell=True)], 0, 480, 270)
    s.evaluate(2.9)
    o.evaluate(2.9)
    report("C2 t=2.9", s, o)
    m = vx.Model.procedural(11, shell=True)
    s, o = pair(4, [m], 0, 640, 360)
    s.evaluate(1.7)
    o.evaluate(1.7)
    report("C4 640x360 t=1.7", s, o, classes=(1, 2, 3), limit=8)
