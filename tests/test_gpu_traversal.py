"""GPU: single-ray traversal (voxanim::traverse -> vxa_traverse, FP64 parity kernel)
against the reference traverse (traversal.cpp:115-252) and the reference's
independent dense-grid DDA oracle (tests/support/oracles.hpp:68-149).

Every TraversalHit field must be bit-identical to the reference (t_hit,
t_enter, t_exit, normal, attribute, the full 16-entry leaf_path array,
path_len) plus the replayed parent node / attribute index and the number of
internal nodes fetched. Rays follow the reference tests' recipe
(test_traversal.cpp:16-34): origins in [-2.5h, 2.5h]^3, 10 % exactly
axis-parallel, plus rays starting on cell boundaries and inside the box.
"""
import numpy as np
import pytest

import paper_1911_06001_b200 as vx
from oracle import ref

pytestmark = pytest.mark.gpu


def make_rays(rng, n, half, depth=3, grid_aligned=0.1):
    rays = np.zeros(n, vx.RAY_DTYPE)
    half = np.asarray(half, np.float64)
    o = rng.uniform(-2.5, 2.5, (n, 3)) * half
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    style = rng.integers(0, 10, n)
    d[style == 0] = np.stack([np.sign(d[style == 0, 0]), 0 * d[style == 0, 0], 0 * d[style == 0, 0]], 1)
    d[style == 1] = np.stack([0 * d[style == 1, 1], np.sign(d[style == 1, 1]), 0 * d[style == 1, 1]], 1)
    xy = style == 2
    nrm = np.hypot(d[xy, 0], d[xy, 1])
    d[xy] = np.stack([d[xy, 0] / nrm, d[xy, 1] / nrm, 0 * nrm], 1)
    # origins snapped onto the cell lattice (half-open boundary conventions)
    snap = rng.random(n) < grid_aligned
    cell = 2 * half / (1 << depth)
    o[snap] = np.round(o[snap] / cell) * cell
    rays["origin"] = o
    rays["direction"] = d
    rays["half_extent"] = half
    return rays


FIELDS = ["hit", "t_hit", "t_enter", "t_exit", "normal_local", "attribute", "attr_index", "node_index", "leaf_path",
          "path_len", "node_fetches"]


def assert_same(ours, theirs):
    for f in FIELDS:
        a, b = ours[f], theirs[f]
        bad = ~np.all(a.reshape(len(a), -1) == b.reshape(len(b), -1), axis=1)
        assert not bad.any(), f"{f}: {int(bad.sum())} of {len(a)} rays differ, first {np.nonzero(bad)[0][:5]}"


def test_random_grids_bit_exact_and_dda(gpu):
    rng = np.random.default_rng(4242)
    for g in range(25):
        depth = int(rng.integers(1, 6))
        fill = float(rng.uniform(0.02, 0.5))
        model = vx.Model.random(1000 + g, depth, fill)
        rmodel = ref.RefModel.random(1000 + g, depth, fill)
        rays = make_rays(rng, 1500, (1.0, 1.0, 1.0), depth)
        assert_same(vx.traverse(model, rays), ref.traverse(rmodel, rays, with_fetches=True))
        # the DDA oracle shares the traversal's conventions for generic rays
        # (the reference's own recipe: no lattice-snapped origins, +0.0 components)
        rays = make_rays(rng, 1500, (1.0, 1.0, 1.0), depth, grid_aligned=0.0)
        rays["direction"] += 0.0
        ours = vx.traverse(model, rays)
        hit, vox, t = ref.dda_random(1000 + g, depth, fill, rays)
        assert (ours["hit"] == hit).all()
        h = hit.astype(bool)
        # leaf_path_to_voxel of our path == DDA voxel
        paths = ours["leaf_path"][h]
        v = np.zeros((h.sum(), 3), np.uint32)
        for lvl in range(depth):
            o = paths[:, lvl].astype(np.uint32)
            v = (v << 1) | np.stack([(o >> 2) & 1, (o >> 1) & 1, o & 1], 1)
        assert (v == vox[h]).all()
        assert np.allclose(ours["t_hit"][h], t[h], rtol=1e-6, atol=1e-9)


def test_anisotropic_bounds(gpu):
    rng = np.random.default_rng(777)
    model, rmodel = vx.Model.random(777, 3, 0.25), ref.RefModel.random(777, 3, 0.25)
    rays = make_rays(rng, 4000, (0.6, 1.7, 0.9), 3)
    assert_same(vx.traverse(model, rays), ref.traverse(rmodel, rays, with_fetches=True))


def test_deep_model_bit_exact(gpu):
    rng = np.random.default_rng(11)
    m = vx.Model.procedural(11, shell=True)
    rm = ref.RefModel.from_bytes(m.serialize())
    rays = make_rays(rng, 20000, (0.7, 1.1, 0.9), 11, grid_aligned=0.2)
    # aim half of the rays at the box so most of them hit the shell
    aim = rng.random(len(rays)) < 0.5
    tgt = rng.uniform(-0.5, 0.5, (aim.sum(), 3)) * np.array([0.7, 1.1, 0.9])
    d = tgt - rays["origin"][aim]
    rays["direction"][aim] = d / np.linalg.norm(d, axis=1, keepdims=True)
    ours = vx.traverse(m, rays)
    assert ours["hit"].mean() > 0.3
    assert_same(ours, ref.traverse(rm, rays, with_fetches=True))


def test_traversal_kats(gpu):
    # reference test_traversal.cpp:96-126
    empty = vx.Model.random(1, 2, 0.0)
    r = np.zeros(1, vx.RAY_DTYPE)
    r["origin"] = (-3, 0.1, 0.1)
    r["direction"] = (1, 0, 0)
    r["half_extent"] = (1, 1, 1)
    assert vx.traverse(empty, r)["hit"][0] == 0
    full = vx.Model.full_cube()
    r["origin"] = (-2, 0.1, 0.1)
    h = vx.traverse(full, r)[0]
    assert h["hit"] == 1 and h["t_hit"] == 1.0
    assert tuple(h["normal_local"]) == (-1.0, 0.0, 0.0)
    assert h["path_len"] == 1 and (h["leaf_path"][0] & 3) == 3  # voxel (., 1, 1)
    assert h["t_enter"] <= h["t_hit"] <= h["t_exit"]
    r["origin"] = (0.5, 0.5, 0.5)
    assert vx.traverse(full, r)[0]["t_hit"] == 0.0
    # parallel ray outside the slab and box behind the origin (test_traversal.cpp:72-80)
    r["origin"] = (0, 5, 0)
    assert vx.traverse(full, r)["hit"][0] == 0
    r["origin"] = (5, 0, 0)
    assert vx.traverse(full, r)["hit"][0] == 0


def test_mirroring_soundness(gpu):
    # reference test_traversal.cpp:152-187: reflected scenes give identical t
    rng = np.random.default_rng(31)
    m = vx.Model.random(31, 3, 0.2)
    rays = make_rays(rng, 400, (1, 1, 1), 3)
    base = vx.traverse(m, rays)
    assert base["hit"].any()
    # reflecting the ray through all three axes and the model is equivalent to
    # the reference's grid reflection; here: reflect the ray only and compare
    # against the reference on the same reflected rays (bit-exact).
    for subset in range(1, 8):
        flip = np.array([(subset >> 2) & 1, (subset >> 1) & 1, subset & 1]) * -2 + 1
        rr = rays.copy()
        rr["origin"] = rays["origin"] * flip
        rr["direction"] = rays["direction"] * flip
        assert_same(vx.traverse(m, rr), ref.traverse(ref.RefModel.random(31, 3, 0.2), rr, with_fetches=True))
