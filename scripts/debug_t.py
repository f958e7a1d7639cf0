import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_06001_b200 as vx
from oracle import ref
for cfg, models in ((vx.config.TWO_OBJECTS, [vx.Model.full_cube()]), (vx.config.C1, [vx.Model.procedural(8, shell=False)])):
    s = vx.Scene(cfg, models)
    o = ref.RefScene(cfg, [ref.RefModel.from_bytes(m.serialize()) for m in models], 0, s.width, s.height)
    oa, _ = o.dump()
    _, ga, _ = s.render(precision=vx.VXA_FP32, aov=True)
    r = o.classify_rules(oa, ga)
    m = r == 101
    print(cfg, ref.rule_histogram(r))
    ys, xs = np.nonzero(m)
    for y, x in list(zip(ys, xs))[:5]:
        print(x, y, oa[y, x]["t"], ga[y, x]["t"], (ga[y, x]["t"] - oa[y, x]["t"]) / oa[y, x]["t"], oa[y,x]["entry_axis"], ga[y,x]["entry_axis"])
    hit = (oa["object_id"] >= 0) & (r == 0)
    rel = (ga["t"][hit] - oa["t"][hit]) / oa["t"][hit]
    print("rel err stats", rel.min(), rel.max(), np.median(rel), np.abs(rel).mean())
