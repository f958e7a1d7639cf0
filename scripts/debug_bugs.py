"""GPU box: explain every pixel the classifier calls a bug (FP32 vs oracle) for a few frames."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_06001_b200 as vx  # noqa: E402
from oracle import ref  # noqa: E402

CASES = [("C2r", vx.config.C2, 10, 2.9, 480, 270), ("C2", vx.config.C2, 10, 1.7, 0, 0), ("C2", vx.config.C2, 10, 3.3, 0, 0),
         ("C4", vx.config.C4, 11, 0.4, 0, 0)]
for name, cfg, depth, t, w, h in CASES:
    m = vx.Model.procedural(depth, shell=True)
    s = vx.Scene(cfg, [m], 0, w, h)
    o = ref.RefScene(cfg, [ref.RefModel.from_bytes(m.serialize())], 0, s.width, s.height)
    s.evaluate(t)
    o.evaluate(t)
    oa, _ = o.dump(threads=ref.hardware_threads())
    _, ga, _ = s.render(precision=vx.VXA_FP32, aov=True)
    r = o.classify_rules(oa, ga)
    ys, xs = np.nonzero(r >= 100)
    print(f"== {name} t={t}: {ref.rule_histogram(r)}", flush=True)
    for y, x in list(zip(ys, xs))[:8]:
        print(o.explain(int(x), int(y), oa[y, x], ga[y, x]), flush=True)
