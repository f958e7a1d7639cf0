"""Golden fixtures (tests/golden/*.npz, generated from the reference by
tests/golden/make_golden.py): the oracles reproduce them on the CPU, the FP64
parity kernel reproduces them on the GPU without any live oracle."""
import os

import numpy as np
import pytest

import paper_1911_06001_b200 as vx
from oracle import ref, restatement

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
import sys  # noqa: E402

sys.path.insert(0, HERE)
import make_golden  # noqa: E402

FRAMES = np.load(os.path.join(HERE, "frames.npz"))
TRAV = np.load(os.path.join(HERE, "traverse.npz"))
TRAV_FIELDS = ("hit", "t_hit", "t_enter", "t_exit", "normal_local", "attribute", "attr_index", "node_index",
               "leaf_path", "path_len", "node_fetches")
FIELDS = ("object_id", "t", "node_index", "attr_index", "level", "entry_axis", "kind", "traversals", "node_fetches")


def same_aov(a, b):
    for k in FIELDS:
        assert (a[k] == b[k]).all(), k
    assert (a["voxel"] == b["voxel"]).all()


def build(name):
    cfg, recipe, seed, w, h, t, culling, sorting = make_golden.SCENES[name]
    models = make_golden.models_for(recipe)
    assert make_golden.model_digest(models).encode() == FRAMES[name + "/models_sha256"].tobytes()
    s = vx.Scene(cfg, models, seed, w, h)
    if t is not None:
        s.evaluate(t)
    return s, models, culling, sorting


@pytest.mark.parametrize("name", sorted(make_golden.SCENES))
def test_restatement_reproduces_golden_frames(name):
    s, models, culling, sorting = build(name)
    objs = [s.get_object(i)[:2] for i in range(s.object_count())]
    recipe = make_golden.SCENES[name][1]
    object_model = list(range(6)) if recipe == "random6" else [0] * len(objs)
    rgb, aov = restatement.render(s.frame_desc(), objs, [m.serialize() for m in models], object_model, culling,
                                  sorting)
    assert (rgb == FRAMES[name + "/rgb"]).all()
    same_aov(aov, FRAMES[name + "/aov"])


@pytest.mark.skipif(not ref.available(), reason="reference oracle not built")
@pytest.mark.parametrize("g", range(8))
def test_reference_reproduces_golden_traversals(g):
    seed, depth, fill = TRAV[f"g{g}/recipe"]
    out = ref.traverse(ref.RefModel.random(int(seed), int(depth), float(fill)), TRAV[f"g{g}/rays"], True)
    exp = TRAV[f"g{g}/hits"]
    for k in TRAV_FIELDS:
        assert (out[k] == exp[k]).all(), k


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(make_golden.SCENES))
def test_fp64_kernel_reproduces_golden_frames(gpu, name):
    s, models, culling, sorting = build(name)
    rgb, aov, _ = s.render(culling, sorting, precision=vx.VXA_FP64, aov=True)
    assert (rgb == FRAMES[name + "/rgb"]).all()
    same_aov(aov, FRAMES[name + "/aov"])


@pytest.mark.gpu
@pytest.mark.parametrize("g", range(8))
def test_fp64_traverse_reproduces_golden(gpu, g):
    seed, depth, fill = TRAV[f"g{g}/recipe"]
    out = vx.traverse(vx.Model.random(int(seed), int(depth), float(fill)), TRAV[f"g{g}/rays"])
    exp = TRAV[f"g{g}/hits"]
    for k in TRAV_FIELDS:
        assert (out[k] == exp[k]).all(), k
