"""GPU: randomized parity sweep. Random model sets (shells, random grids, dense
spheres, full cubes), random rigid transforms (config RANDOM), random look-at
cameras -- far, near, inside an instance, any orientation and field of view --
and random culling/sorting options. FP64 kernel: bit-exact with the reference
per pixel (image, hit, node, attribute, level, voxel, t, counts); FP32 kernel:
hits identical except classified slab-test ties (tests/test_gpu_parity.py)."""
import os

import numpy as np
import pytest

import paper_1911_06001_b200 as vx
from test_gpu_parity import check_fp32, check_fp64, pair

pytestmark = pytest.mark.gpu


def random_models(rng):
    out = []
    for _ in range(int(rng.integers(3, 6))):
        kind = rng.integers(0, 4)
        if kind == 0:
            out.append(vx.Model.procedural(int(rng.integers(3, 9)), shell=bool(rng.integers(0, 2))))
        elif kind == 1:
            out.append(vx.Model.random(int(rng.integers(0, 1 << 30)), int(rng.integers(2, 7)), float(rng.uniform(0.01, 0.6))))
        elif kind == 2:
            out.append(vx.Model.dense_sphere(int(rng.integers(2, 6))))
        else:
            out.append(vx.Model.full_cube())
    return out


def unit(rng):
    v = rng.normal(size=3)
    return v / np.linalg.norm(v)


# VOXANIM_FUZZ_SEEDS=N widens the sweep (a soak run); 64 by default. Seeds 96, 174
# and 177 found (in a 400-seed soak) spheres wholly behind the camera that the
# reference's loose sphere test counts as hit while the tile cone dropped them.
SEEDS = sorted(set(range(int(os.environ.get("VOXANIM_FUZZ_SEEDS", "64")))) | {96, 174, 177})


@pytest.mark.parametrize("seed", SEEDS)
def test_random_scene_random_camera(gpu, seed):
    rng = np.random.default_rng(1000 + seed)
    models = random_models(rng)
    s, o = pair(vx.config.RANDOM, models, seed=int(rng.integers(0, 1 << 30)), w=128, h=96)
    if rng.uniform() < 0.15:
        # inside (or at the surface of) an instance
        _, tf, _ = s.get_object(int(rng.integers(0, len(models))))
        pos = np.array(tf[9:12]) + rng.uniform(-0.3, 0.3, 3)
    else:
        pos = unit(rng) * rng.uniform(3.0, 14.0)
    if rng.uniform() < 0.7:  # look at an instance
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
    o_aov, o_img = check_fp64(s, o, culling, sorting)
    check_fp32(s, o, o_aov, o_img, culling, sorting, max_tie_frac=0.02)
