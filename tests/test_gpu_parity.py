"""GPU parity: the CUDA frame against the reference CPU renderer (oracle/_ref).

FP64 parity kernel: bit-exact image, hit object, leaf-parent node, attribute
index, level, voxel and t for every pixel.
FP32 production kernel: every pixel whose hit differs from the oracle must be
a documented slab-test tie (oracle/ref_harness.cpp classify_pixel); where the
hit agrees, t must be within 1e-6 relative (floor 1e-6 absolute) and RGB
within +-1 LSB per channel.
"""
import numpy as np
import pytest

import paper_1911_06001_b200 as vx
from oracle import ref

pytestmark = pytest.mark.gpu

T_REL = 1e-6


def pair(cfg, models, seed=0, w=0, h=0):
    """(product scene, oracle scene) built from the same models (oracle side via .svo bytes)."""
    rmodels = [ref.RefModel.from_bytes(m.serialize()) for m in models]
    s = vx.Scene(cfg, models, seed, w, h)
    o = ref.RefScene(cfg, rmodels, seed, s.width, s.height)
    return s, o


def check_fp64(s, o, culling=True, sorting=True):
    o_aov, o_rgb = o.dump(culling, sorting)
    o_img, o_st = o.render(culling, sorting)
    assert (o_rgb == o_img).all()
    rgb, aov, st = s.render(culling, sorting, precision=vx.VXA_FP64, aov=True)
    assert (rgb == o_img).all(), f"{int((rgb != o_img).any(axis=2).sum())} pixels differ"
    for f in ("object_id", "node_index", "attr_index", "level", "entry_axis", "t", "kind", "traversals",
              "node_fetches"):
        bad = aov[f] != o_aov[f]
        assert not bad.any(), f"{f}: {int(bad.sum())} pixels differ"
    assert (aov["voxel"] == o_aov["voxel"]).all()
    for k in ("rays", "sphere_tests", "svo_traversals", "pixels_reused"):
        assert st[k] == o_st[k], k
    o.last_stats = o_st
    return o_aov, o_img


def check_fp32(s, o, o_aov, o_img, culling=True, sorting=True, max_tie_frac=5e-3, max_kind_frac=1e-3):
    """FP32 production kernel vs the oracle. Every differing pixel must be a
    documented tie (oracle/ref_harness.cpp classify_rule); matching hits within the
    t tolerance and +-1 LSB. FP32 FrameStats semantics: rays and sphere_tests are
    counted on the host (pixels x objects) and equal the reference's; the FP32
    sphere test is conservative (a margin of 1e-5 relative), so it may admit a
    grazed sphere the FP64 test rejects, and its t_boundary is lowered by the same
    margin (a skip can only come later) -- svo_traversals is not below the
    reference's (up to a tie or two) and exceeds it by at most 1e-4 relative (+8);
    HitKind may read MultiSphere for SingleSphere on such pixels (full-size frames:
    <= 1e-5 of the pixels)."""
    rgb, aov, st = s.render(culling, sorting, precision=vx.VXA_FP32, aov=True)
    # the production instantiation (no AOV stores) renders the same image as the
    # AOV one the classifier checks
    prod = s.render(culling, sorting, precision=vx.VXA_FP32)[0]
    assert (prod == rgb).all(), f"{int((prod != rgb).any(axis=2).sum())} pixels differ between FP32 kernels"
    rules = o.classify_rules(o_aov, aov, T_REL)
    hist = ref.rule_histogram(rules)
    n_hit = max(1, int((o_aov["object_id"] >= 0).sum()))
    bugs = int((rules == ref.RULE_BUG).sum())
    t_bad = int((rules == ref.RULE_T_OUT).sum())
    assert bugs == 0, f"{bugs} unexplained FP32 mismatches {hist}"
    assert t_bad == 0, f"{t_bad} pixels with t outside the tolerance {hist}"
    ties = int(((rules > 0) & (rules < 100)).sum())
    assert ties <= max_tie_frac * n_hit + 2, f"{ties} ties of {n_hit} hits {hist}"
    same = rules == 0
    diff = np.abs(rgb.astype(int) - o_img.astype(int)).max(axis=2)
    assert (diff[same] <= 1).all(), "RGB outside +-1 LSB on matching pixels"
    o_st = getattr(o, "last_stats", None)
    if o_st is not None:
        assert st["rays"] == o_st["rays"] and st["sphere_tests"] == o_st["sphere_tests"]
        extra = st["svo_traversals"] - o_st["svo_traversals"]
        assert -2 - 1e-5 * o_st["svo_traversals"] <= extra <= 1e-4 * o_st["svo_traversals"] + 8, \
            (st["svo_traversals"], o_st["svo_traversals"])
        kind_bad = int(((aov["kind"] != o_aov["kind"]) & same).sum())
        assert kind_bad <= max_kind_frac * rules.size + 2, kind_bad
    return ties, n_hit, hist


def test_sorted_tracing_scene(gpu):
    s, o = pair(vx.config.SORTED_TRACING, [vx.Model.full_cube()])
    o_aov, o_img = check_fp64(s, o)
    check_fp32(s, o, o_aov, o_img)


def test_two_objects(gpu):
    s, o = pair(vx.config.TWO_OBJECTS, [vx.Model.full_cube()])
    o_aov, o_img = check_fp64(s, o)
    check_fp32(s, o, o_aov, o_img)


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_random_scenes_all_option_combinations(gpu, seed):
    models = [vx.Model.random(100 * seed + k, 2 + (k % 3), 0.3) for k in range(6)]
    s, o = pair(vx.config.RANDOM, models, seed)
    for culling in (True, False):
        for sorting in (True, False):
            o_aov, o_img = check_fp64(s, o, culling, sorting)
            check_fp32(s, o, o_aov, o_img, culling, sorting)


def test_c1_full_size(gpu):
    s, o = pair(vx.config.C1, [vx.Model.procedural(8, shell=False)])
    o_aov, o_img = check_fp64(s, o)
    check_fp32(s, o, o_aov, o_img)


@pytest.mark.parametrize("t", [0.0, 0.5, 1.3, 2.9])
def test_c2_animated_frames_reduced(gpu, t):
    s, o = pair(vx.config.C2, [vx.Model.procedural(10, shell=True)], w=480, h=270)
    s.evaluate(t)
    o.evaluate(t)
    o_aov, o_img = check_fp64(s, o)
    check_fp32(s, o, o_aov, o_img)


def test_c4_reduced(gpu):
    s, o = pair(vx.config.C4, [vx.Model.procedural(11, shell=True)], w=640, h=360)
    for t in (0.0, 1.7):
        s.evaluate(t)
        o.evaluate(t)
        o_aov, o_img = check_fp64(s, o)
        check_fp32(s, o, o_aov, o_img)


def mixed_node_model():
    """A hand-built (non-canonical) model: the root holds a leaf voxel next to an
    internal child -- valid for the reference (svo.cpp validate) but not for the
    compact node words, so the general words + side array are exercised."""
    import struct

    nodes = [(1, 0, 0b00000011, 0b00000001), (0, 1, 0xFF, 0xFF)]
    attrs = [(200, 40, 40, 255)] + [(40 + 20 * k, 200 - 10 * k, 90, 255) for k in range(8)]
    data = b"SVOA" + struct.pack("<IIII", 1, 2, len(nodes), len(attrs))
    for cb, ab, v, l in nodes:
        data += struct.pack("<IIBBH", cb, ab, v, l, 0)
    for a in attrs:
        data += bytes(a)
    return vx.Model.from_bytes(data)


def test_mixed_node_model(gpu):
    m = mixed_node_model()
    s, o = pair(vx.config.TWO_OBJECTS, [m])
    o_aov, o_img = check_fp64(s, o)
    assert (o_aov["object_id"] >= 0).sum() > 100
    check_fp32(s, o, o_aov, o_img)


@pytest.mark.parametrize("words", ["wide", "compact"])
def test_node_word_formats_agree(gpu, words, monkeypatch):
    """C4 reduced with the general 8-byte words forced (VOXANIM_NODE_WORDS=wide)
    and with the compact words: both parity-clean against the oracle."""
    monkeypatch.setenv("VOXANIM_NODE_WORDS", words)
    s, o = pair(vx.config.C4, [vx.Model.procedural(9, shell=True)], w=320, h=180)
    s.evaluate(0.9)
    o.evaluate(0.9)
    o_aov, o_img = check_fp64(s, o)
    check_fp32(s, o, o_aov, o_img)


@pytest.mark.parametrize("cfg,t", [(vx.config.C2, 1.7), (vx.config.C4, 2.3)])
def test_full_size_frame(gpu, cfg, t):
    """BASELINE configurations at their full resolution (C2 1920x1080 depth 10,
    C4 3840x2160 with 64 depth-11 instances): FP64 bit-exact, FP32 ties only."""
    depth = 10 if cfg == vx.config.C2 else 11
    s, o = pair(cfg, [vx.Model.procedural(depth, shell=True)])
    s.evaluate(t)
    o.evaluate(t)
    o_aov, o_img = check_fp64(s, o)
    # tie caps: 3x the largest rate measured over full-size frames (profiles/fp32_evidence_r2.json:
    # C2 <= 0.017 %, C4 <= 0.165 % of hit pixels; the rate scales with t 2^depth / scale,
    # the FP32 resolution of a plane position relative to the voxel size)
    cap = 5e-4 if cfg == vx.config.C2 else 5e-3
    ties, n_hit, hist = check_fp32(s, o, o_aov, o_img, max_tie_frac=cap, max_kind_frac=1e-5)
    print(f"config {cfg}: {n_hit} hit pixels, {ties} FP32 ties ({100.0 * ties / n_hit:.4f} %) {hist}")


def test_axis_aligned_camera_zero_direction_rays(gpu):
    """Odd resolution on the z axis with identity transforms: the middle row and
    column carry exactly-zero local direction components (traversal.cpp:19-21,
    135-140 zero-direction convention)."""
    s, o = pair(vx.config.AXIS_ALIGNED, [vx.Model.procedural(6, shell=False), vx.Model.random(9, 4, 0.3)])
    o_aov, o_img = check_fp64(s, o)
    assert (o_aov["object_id"][50, :] >= 0).sum() > 10  # the zero-direction row hits
    # the centre row/column run exactly along cell faces: ties by construction
    check_fp32(s, o, o_aov, o_img, max_tie_frac=0.02)


def test_many_instances_overflow_the_tile_list(gpu):
    """200 instances: tiles whose cone meets more than 64 instances fall back to
    the per-ray pass over every instance; results stay parity-clean."""
    models = [vx.Model.procedural(6, shell=True), vx.Model.random(4, 4, 0.2)]
    s, o = pair(vx.config.MANY, models, seed=3)
    for culling, sorting in ((True, True), (True, False)):
        o_aov, o_img = check_fp64(s, o, culling, sorting)
        check_fp32(s, o, o_aov, o_img, culling, sorting)


def test_stacked_instances_overflow_tile_lists(gpu):
    """96 instances stacked along the view axis: the tiles around the axis meet
    all 96 (> the 64-entry tile list), so they take the per-ray fallback pass
    over every instance, next to list tiles elsewhere in the frame."""
    models = [vx.Model.procedural(6, shell=True), vx.Model.random(9, 5, 0.1)]
    s, o = pair(vx.config.STACKED, models, seed=5)
    for culling, sorting in ((True, True), (True, False), (False, True)):
        o_aov, o_img = check_fp64(s, o, culling, sorting)
        check_fp32(s, o, o_aov, o_img, culling, sorting)


def test_crowd_reduced(gpu):
    """The crowd configuration with 512 animated
    instances at 640x360, two animation times."""
    models = [vx.Model.procedural(7, shell=True)]
    s, o = pair(vx.config.CROWD, models, seed=512, w=640, h=360)
    for t in (0.4, 2.3):
        s.evaluate(t)
        o.evaluate(t)
        o_aov, o_img = check_fp64(s, o)
        check_fp32(s, o, o_aov, o_img)


def test_deep_model_depth_12(gpu):
    """A depth-12 shell (21 M nodes, 44 M attributes -- past the compact words'
    2^24 range, so the general words run at scale): FP64 per-ray bit-exact vs the
    reference, and a frame through both kernels."""
    m = vx.Model.procedural(12, shell=True)
    rm = ref.RefModel.from_bytes(m.serialize())
    rng = np.random.default_rng(13)
    n = 4000
    rays = np.zeros(n, vx.RAY_DTYPE)
    rays["origin"] = rng.uniform(-2, 2, (n, 3))
    tgt = rng.uniform(-0.3, 0.3, (n, 3))
    d = tgt - rays["origin"]
    rays["direction"] = d / np.linalg.norm(d, axis=1, keepdims=True)
    rays["half_extent"] = (0.5, 0.5, 0.5)
    ours, theirs = vx.traverse(m, rays), ref.traverse(rm, rays, with_fetches=True)
    assert ours["hit"].mean() > 0.5
    for k in ("hit", "t_hit", "leaf_path", "path_len", "node_index", "attr_index", "node_fetches"):
        assert (ours[k] == theirs[k]).all(), k
    s, o = pair(vx.config.C1, [m], w=128, h=128)
    o_aov, o_img = check_fp64(s, o)
    check_fp32(s, o, o_aov, o_img)


def _rotation(seed):
    q = np.random.default_rng(seed).normal(size=4)
    w, x, y, z = q / np.linalg.norm(q)
    return [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w),
            2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w),
            2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]


@pytest.mark.parametrize("seed", [1, 2])
def test_camera_inside_an_instance(gpu, seed):
    """The camera inside an instance's box and bounding sphere (ray origins inside
    the root cell: negative entry parameters, hits on the shell's inner side),
    next to an ordinary instance; every culling/sorting option."""
    models = [vx.Model.procedural(7, shell=True), vx.Model.random(seed, 5, 0.05)]
    s, o = pair(vx.config.TWO_OBJECTS, models)
    for sc in (s, o):
        sc.set_object(0, _rotation(seed) + [0.1, -0.05, 7.8] + [3.0, 2.5, 3.5], True)
        sc.set_object(1, _rotation(seed + 10) + [0.3, 0.2, 6.9] + [0.8, 0.8, 0.8], True)
    for culling, sorting in ((True, True), (False, False), (True, False)):
        o_aov, o_img = check_fp64(s, o, culling, sorting)
        assert (o_aov["object_id"] >= 0).mean() > 0.5  # the inner shell fills the view
        check_fp32(s, o, o_aov, o_img, culling, sorting)


def test_degenerate_scales(gpu):
    """Zero and negative scale components (rejected by the scene loader but
    reachable through the API): the reference finds no hit in such a box; both
    kernels agree with it (the FP32 kernel skips the instance)."""
    models = [vx.Model.procedural(6, shell=True), vx.Model.random(3, 4, 0.4)]
    s, o = pair(vx.config.TWO_OBJECTS, models)
    for sc in (s, o):
        sc.set_object(0, _rotation(5) + [-1.0, 0.0, 0.0] + [2.0, 0.0, 2.0], True)
        sc.set_object(1, _rotation(6) + [1.5, 0.2, 0.0] + [-1.5, 1.5, 1.5], True)
    for culling, sorting in ((True, True), (False, True)):
        o_aov, o_img = check_fp64(s, o, culling, sorting)
        rgb, aov, _ = s.render(culling, sorting, precision=vx.VXA_FP32, aov=True)
        assert (rgb == o_img).all()


def test_super_tile_list_overflow(gpu):
    """1500 instances in a 64x36 frame: one super-tile whose cone meets more than
    the 1024-entry super-tile list, so its tiles fall back to testing every
    instance (the pre-pass overflow path); 8x4 tile lists then overflow too."""
    models = [vx.Model.procedural(5, shell=True)]
    s, o = pair(vx.config.CROWD, models, seed=1500, w=64, h=36)
    for t in (0.0, 1.7):
        s.evaluate(t)
        o.evaluate(t)
        o_aov, o_img = check_fp64(s, o)
        check_fp32(s, o, o_aov, o_img)


def _depth_first_layout(svo: bytes) -> bytes:
    """The same octree with nodes numbered depth-first (each node's children
    allocated as one contiguous block when the node is visited, so children
    still follow their parent) and attributes renumbered in that order: a
    valid .svo that is not in the reference builder's breadth-first order."""
    import struct
    depth, nn, na = struct.unpack_from("<III", svo, 8)
    recs = [struct.unpack_from("<IIBB", svo, 20 + 12 * i) for i in range(nn)]
    attrs = [svo[20 + 12 * nn + 4 * k: 24 + 12 * nn + 4 * k] for k in range(na)]
    new_of = {0: 0}
    out_nodes, out_attrs = [None] * nn, []
    next_free = 1

    def visit(old):
        nonlocal next_free
        cb, ab, valid, leaf = recs[old]
        internal = valid & ~leaf & 0xFF
        kids = bin(internal).count("1")
        leaves = bin(valid & leaf).count("1")
        new_cb = next_free if kids else 0
        next_free += kids
        new_ab = len(out_attrs) if leaves else 0
        out_attrs.extend(attrs[ab:ab + leaves])
        out_nodes[new_of[old]] = (new_cb, new_ab, valid, leaf)
        for k in range(kids):
            new_of[cb + k] = new_cb + k
        for k in range(kids):
            visit(cb + k)

    visit(0)
    body = b"".join(struct.pack("<IIBBxx", *r) for r in out_nodes)
    return svo[:20] + body + b"".join(out_attrs)


def test_depth_first_node_layout(gpu):
    """A model whose nodes are not in breadth-first order (any order with
    children after their parent is a valid .svo): both kernels render it like
    the reference renders the same bytes."""
    import sys
    sys.setrecursionlimit(10000)
    for base in (vx.Model.random(31, 5, 0.15), vx.Model.procedural(6, shell=True)):
        dfs = _depth_first_layout(base.serialize())
        assert dfs != base.serialize()
        m = vx.Model.from_bytes(dfs)
        assert m.violations() == 0
        s, o = pair(vx.config.RANDOM, [m, vx.Model.full_cube()], seed=8)
        for culling, sorting in ((True, True), (False, False)):
            o_aov, o_img = check_fp64(s, o, culling, sorting)
            check_fp32(s, o, o_aov, o_img, culling, sorting)
