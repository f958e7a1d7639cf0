"""Regenerates the golden fixtures from the REFERENCE (oracle/_ref, compiled from
/root/reference by oracle/Makefile). Run here, not on the GPU box:

    python tests/golden/make_golden.py

frames.npz  per-pixel AOVs + RGB of the reference render (shade_pixel replay
            checked against render_frame) for small scenes: random 6-object
            scenes under all four culling/sorting options, the reference test
            layouts, C1/C2/C4 at reduced resolution (animated where the config is).
traverse.npz  reference traverse() on random local rays against random grids
            (seeded like tests/support/oracles.hpp), incl. axis-parallel rays.
Models are not stored: the builders are byte-identical to the reference's
(tests/test_builder.py); their SHA-256 is stored to catch drift.
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_1911_06001_b200 as vx  # noqa: E402  (host-side model builders only)
from oracle import ref  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# name -> (config, model recipe, seed, width, height, time, culling, sorting)
SCENES = {
    "random_cs": (5, "random6", 7, 0, 0, None, True, True),
    "random_c": (5, "random6", 7, 0, 0, None, True, False),
    "random_s": (5, "random6", 7, 0, 0, None, False, True),
    "random_none": (5, "random6", 7, 0, 0, None, False, False),
    "sorted_tracing": (6, "cube", 0, 0, 0, None, True, True),
    "two_objects": (7, "cube", 0, 0, 0, None, True, True),
    "c1_128": (1, "solid7", 0, 128, 128, None, True, True),
    "c2_160_t2.2": (2, "shell8", 0, 160, 90, 2.2, True, True),
    "c4_192_t1.3": (4, "shell7", 0, 192, 108, 1.3, True, True),
}


def models_for(recipe):
    if recipe == "random6":
        return [vx.Model.random(50 + k, 2 + k % 3, 0.3) for k in range(6)]
    if recipe == "cube":
        return [vx.Model.full_cube()]
    if recipe == "solid7":
        return [vx.Model.procedural(7, shell=False)]
    if recipe == "shell8":
        return [vx.Model.procedural(8, shell=True)]
    if recipe == "shell7":
        return [vx.Model.procedural(7, shell=True)]
    raise KeyError(recipe)


def model_digest(models):
    h = hashlib.sha256()
    for m in models:
        h.update(m.serialize())
    return h.hexdigest()


def make_frames():
    out = {}
    for name, (cfg, recipe, seed, w, h, t, culling, sorting) in SCENES.items():
        models = models_for(recipe)
        o = ref.RefScene(cfg, [ref.RefModel.from_bytes(m.serialize()) for m in models], seed, w, h)
        if t is not None:
            o.evaluate(t)
        aov, rgb = o.dump(culling, sorting)
        img, _ = o.render(culling, sorting)
        assert (img == rgb).all(), name
        out[name + "/aov"] = aov
        out[name + "/rgb"] = rgb
        out[name + "/models_sha256"] = np.frombuffer(model_digest(models).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "frames.npz"), **out)


def make_traverse():
    rng = np.random.default_rng(2024)
    out = {}
    for g in range(8):
        depth = 1 + g % 5
        fill = 0.05 + 0.05 * g
        seed = 900 + g
        n = 400
        rays = np.zeros(n, ref.RAY_DTYPE)
        rays["origin"] = rng.uniform(-2.5, 2.5, (n, 3))
        d = rng.normal(size=(n, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        ax = rng.integers(0, 10, n)
        d[ax == 0] = np.stack([np.sign(d[ax == 0, 0]), np.zeros((ax == 0).sum()), np.zeros((ax == 0).sum())], 1)
        rays["direction"] = d
        rays["half_extent"] = (1.0, 1.0, 1.0)
        hits = ref.traverse(ref.RefModel.random(seed, depth, fill), rays, with_fetches=True)
        out[f"g{g}/rays"] = rays
        out[f"g{g}/hits"] = hits
        out[f"g{g}/recipe"] = np.array([seed, depth, fill])
    np.savez_compressed(os.path.join(HERE, "traverse.npz"), **out)


if __name__ == "__main__":
    make_frames()
    make_traverse()
    for f in ("frames.npz", "traverse.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)))
