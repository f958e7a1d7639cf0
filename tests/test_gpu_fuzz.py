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
from oracle import ref
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


def _random_camera(rng, s):
    _, tf, _ = s.get_object(int(rng.integers(0, s.object_count())))
    at = np.array(tf[9:12]) + rng.uniform(-1.0, 1.0, 3)
    pos = at + unit(rng) * rng.uniform(0.5, 9.0)
    up = unit(rng)
    fwd = (at - pos) / np.linalg.norm(at - pos)
    if np.linalg.norm(np.cross(fwd, up)) < 0.1:
        up = np.array([0.0, 1.0, 0.0]) if abs(fwd[1]) < 0.9 else np.array([1.0, 0.0, 0.0])
    return pos.tolist(), at.tolist(), up.tolist(), float(rng.uniform(25.0, 100.0))


SEEDS_MANY = range(int(os.environ.get("VOXANIM_FUZZ_SEEDS_MANY", "12")))


@pytest.mark.parametrize("seed", SEEDS_MANY)
def test_many_instances_random_camera(gpu, seed):
    """200 instances (config MANY: the super-tile culling pre-pass runs) seen
    from random cameras, in and around the crowd."""
    rng = np.random.default_rng(5000 + seed)
    models = [vx.Model.procedural(int(rng.integers(4, 7)), shell=True), vx.Model.random(seed, 4, 0.3)]
    s, o = pair(vx.config.MANY, models, seed=seed, w=160, h=120)
    cam = _random_camera(rng, s)
    for sc in (s, o):
        sc.set_camera(*cam)
    o_aov, o_img = check_fp64(s, o)
    check_fp32(s, o, o_aov, o_img, max_tie_frac=0.02)


SEEDS_HBO = range(int(os.environ.get("VOXANIM_FUZZ_SEEDS_HBO", "8")))


@pytest.mark.parametrize("seed", SEEDS_HBO)
def test_hit_buffer_random_sequences(gpu, seed):
    """Random scenes and cameras, 12 frames with the hit buffer: objects moved or
    touched at random, the camera made dirty at random. FP64: image, FrameStats
    and every record equal the reference's with its own HitBuffer."""
    rng = np.random.default_rng(7000 + seed)
    models = random_models(rng)
    s, o = pair(vx.config.RANDOM, models, seed=int(rng.integers(0, 1 << 30)), w=96, h=64)
    cam = _random_camera(rng, s)
    for sc in (s, o):
        sc.set_camera(*cam)
    hbo, rhbo = vx.HitBuffer(96, 64), ref.RefHitBuffer(96, 64)
    for frame in range(12):
        for _ in range(int(rng.integers(0, 3))):
            i = int(rng.integers(0, s.object_count()))
            _, tf, _ = s.get_object(i)
            if rng.uniform() < 0.5:
                tf[9:12] = (np.array(tf[9:12]) + rng.uniform(-0.3, 0.3, 3)).tolist()
            for sc in (s, o):
                sc.set_object(i, tf, True)
        if rng.uniform() < 0.2:
            for sc in (s, o):
                sc.set_camera_dirty(True)
        a, _, st = s.render(precision=vx.VXA_FP64, hbo=hbo)
        r, rst = o.render(hbo=rhbo)
        assert (a == r).all(), frame
        for k in ("pixels_reused", "svo_traversals", "sphere_tests"):
            assert st[k] == rst[k], (frame, k)
        ours, theirs = hbo.records(), rhbo.records()
        for f in ("color", "normal", "t", "object_id", "kind"):
            assert (ours[f] == theirs[f]).all(), (frame, f)
        for sc in (s, o):
            sc.mark_clean()


SEEDS_BUILD = range(int(os.environ.get("VOXANIM_FUZZ_SEEDS_BUILD", "8")))


@pytest.mark.parametrize("seed", SEEDS_BUILD)
def test_device_builder_random_grids(gpu, seed):
    """vxa_build_model on random grids (depth 1-7, fills from empty to full,
    clustered or uniform, every colour mode): byte-identical to the reference."""
    rng = np.random.default_rng(9000 + seed)
    depth = int(rng.integers(1, 8))
    n = 1 << depth
    if rng.uniform() < 0.5:
        bits = rng.random(n ** 3) < rng.uniform(0.0, 1.0) ** 3
    else:  # clusters: a few random boxes
        g = np.zeros((n, n, n), bool)
        for _ in range(int(rng.integers(1, 6))):
            lo = rng.integers(0, n, 3)
            hi = lo + rng.integers(1, n + 1, 3)
            g[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = True
        bits = g.ravel()
    pad = (-bits.size) % 64
    b = np.concatenate([bits, np.zeros(pad, bool)]).reshape(-1, 64)
    words = (b.astype(np.uint64) << np.arange(64, dtype=np.uint64)).sum(axis=1, dtype=np.uint64)
    mode = int(rng.integers(0, 3))
    rgba = int(rng.integers(0, 1 << 32))
    ours = vx.Model.from_grid(words, depth, mode, rgba, device=True).serialize()
    assert ours == ref.RefModel.from_grid(words, depth, mode, rgba).serialize(), (depth, mode)


SEEDS_SVO = range(int(os.environ.get("VOXANIM_FUZZ_SEEDS_SVO", "8")))


@pytest.mark.parametrize("seed", SEEDS_SVO)
def test_svo_stream_random_corruption(gpu, seed):
    """vxa_upload_svo on randomly corrupted .svo streams (byte flips, truncation,
    extension): whenever the reference's deserialize() rejects a stream, so do we,
    with its SvoFormatErrorCode class and message; a stream it accepts we accept
    too unless the reference's validate() flags it (the GPU needs a valid model)."""
    import ctypes as C

    rng = np.random.default_rng(11000 + seed)
    good = bytearray(vx.Model.random(int(rng.integers(0, 1 << 30)), int(rng.integers(1, 5)), 0.4).serialize())
    lib, ctx = vx.vxa(), vx.context()
    for _ in range(40):
        data = bytearray(good)
        op = rng.integers(0, 3)
        if op == 0:
            for _ in range(int(rng.integers(1, 4))):
                data[int(rng.integers(0, len(data)))] = int(rng.integers(0, 256))
        elif op == 1:
            data = data[:int(rng.integers(0, len(data)))]
        else:
            data += bytes(int(rng.integers(1, 9)))
        data = bytes(data)
        h, code = C.c_uint32(), C.c_int32()
        rc = lib.vxa_upload_svo(ctx, data, len(data), C.byref(h), C.byref(code))
        try:
            rm = ref.RefModel.from_bytes(data)
            ref_err = None
        except RuntimeError as e:
            rm, ref_err = None, str(e)
        if ref_err is not None:
            assert rc == 2 and code.value >= 0, (ref_err, rc)
            assert lib.vxa_last_error().decode() == ref_err
        elif rc == 0:
            lib.vxa_release_model(ctx, h.value)
        else:
            assert code.value == -1 and rm.violations() > 0, lib.vxa_last_error().decode()
