"""Debug helper (not a test): print FP32-vs-oracle mismatch breakdowns on the GPU box."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1911_06001_b200 as vx
from oracle import ref


def report(name, s, o, culling=True, sorting=True, limit=6):
    o_aov, _ = o.dump(culling, sorting)
    _, aov, _ = s.render(culling, sorting, precision=vx.VXA_FP32, aov=True)
    cls = o.classify(o_aov, aov, 1e-6)
    print(f"== {name}: hits {(o_aov['object_id']>=0).sum()} match {(cls==0).sum()} tie {(cls==1).sum()} "
          f"bug {(cls==2).sum()} t_out {(cls==3).sum()}")
    for c in (2, 3):
        ys, xs = np.nonzero(cls == c)
        for y, x in list(zip(ys, xs))[:limit]:
            print(o.explain(int(x), int(y), o_aov[y, x], aov[y, x]))
            if c == 3:
                print("   rel err", abs(o_aov[y, x]['t'] - aov[y, x]['t']) / max(1, abs(o_aov[y, x]['t'])))


def pair(cfg, models, seed=0, w=0, h=0):
    rmodels = [ref.RefModel.from_bytes(m.serialize()) for m in models]
    s = vx.Scene(cfg, models, seed, w, h)
    o = ref.RefScene(cfg, rmodels, seed, s.width, s.height)
    return s, o


models = [vx.Model.random(100 * 2 + k, 2 + (k % 3), 0.3) for k in range(6)]
s, o = pair(5, models, 2)
report("random seed 2", s, o)
m = vx.Model.procedural(7, shell=True)
s, o = pair(4, [m], 0, 192, 108)
s.evaluate(1.25); o.evaluate(1.25)
report("C4 depth7 192x108", s, o)
