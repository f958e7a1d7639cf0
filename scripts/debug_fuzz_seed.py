"""GPU box: explain the FP32 pixels the classifier rejects for one fuzz seed."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1911_06001_b200 as vx  # noqa: E402
from oracle import ref  # noqa: E402
from test_gpu_fuzz import random_models, unit  # noqa: E402
from test_gpu_parity import pair  # noqa: E402

for seed in [int(a) for a in sys.argv[1:]]:
    rng = np.random.default_rng(1000 + seed)
    models = random_models(rng)
    s, o = pair(vx.config.RANDOM, models, seed=int(rng.integers(0, 1 << 30)), w=128, h=96)
    if rng.uniform() < 0.15:
        _, tf, _ = s.get_object(int(rng.integers(0, len(models))))
        pos = np.array(tf[9:12]) + rng.uniform(-0.3, 0.3, 3)
    else:
        pos = unit(rng) * rng.uniform(3.0, 14.0)
    if rng.uniform() < 0.7:
        _, tf, _ = s.get_object(int(rng.integers(0, len(models))))
        at = np.array(tf[9:12]) + rng.uniform(-0.5, 0.5, 3)
    else:
        at = rng.uniform(-2.0, 2.0, 3)
    if np.linalg.norm(at - pos) < 0.5:
        at = pos + unit(rng)
    fwd = (at - pos) / np.linalg.norm(at - pos)
    up = unit(rng)
    if np.linalg.norm(np.cross(fwd, up)) < 0.1:
        up = np.array([0.0, 1.0, 0.0]) if abs(fwd[1]) < 0.9 else np.array([1.0, 0.0, 0.0])
    fov = float(rng.uniform(20.0, 100.0))
    for sc in (s, o):
        sc.set_camera(pos.tolist(), at.tolist(), up.tolist(), fov)
    culling, sorting = bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
    oa, _ = o.dump(culling, sorting)
    _, ga, _ = s.render(culling, sorting, precision=vx.VXA_FP32, aov=True)
    r = o.classify_rules(oa, ga)
    print(f"== seed {seed}: culling {culling} sorting {sorting} fov {fov:.1f} pos {pos} {ref.rule_histogram(r)}")
    ys, xs = np.nonzero(r >= 100)
    for y, x in list(zip(ys, xs))[:6]:
        print(o.explain(int(x), int(y), oa[y, x], ga[y, x]), flush=True)
