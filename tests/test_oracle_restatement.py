"""CPU: the plain-C restatement (oracle/voxanim_oracle.c) is bit-exact with the
reference itself (oracle/_ref) on the per-pixel AOVs and the image, for every
culling / sorting option and for the benchmark layouts (reduced sizes)."""
import numpy as np
import pytest

import paper_1911_06001_b200 as vx
from oracle import ref, restatement

FIELDS = ("object_id", "t", "node_index", "attr_index", "level", "entry_axis", "kind", "traversals", "node_fetches")


def compare(cfg, models, object_model, seed=0, w=0, h=0, t=None, culling=True, sorting=True):
    s = vx.Scene(cfg, models, seed, w, h)
    o = ref.RefScene(cfg, [ref.RefModel.from_bytes(m.serialize()) for m in models], seed, s.width, s.height)
    if t is not None:
        s.evaluate(t)
        o.evaluate(t)
    f = s.frame_desc()
    objs = []
    for i in range(s.object_count()):
        oid, tf, _ = s.get_object(i)
        objs.append((oid, tf))
    rgb, aov = restatement.render(f, objs, [m.serialize() for m in models], object_model, culling, sorting)
    o_aov, o_rgb = o.dump(culling, sorting)
    assert (rgb == o_rgb).all()
    for k in FIELDS:
        assert (aov[k] == o_aov[k]).all(), k
    assert (aov["voxel"] == o_aov["voxel"]).all()
    return aov


@pytest.mark.parametrize("culling,sorting", [(True, True), (True, False), (False, True), (False, False)])
def test_random_scene_all_options(culling, sorting):
    models = [vx.Model.random(50 + k, 2 + k % 3, 0.3) for k in range(6)]
    compare(vx.config.RANDOM, models, list(range(6)), seed=7, culling=culling, sorting=sorting)


def test_reference_test_layouts():
    cube = vx.Model.full_cube()
    compare(vx.config.SORTED_TRACING, [cube], [0] * 4)
    compare(vx.config.TWO_OBJECTS, [cube], [0] * 2)


def test_c1_and_c4_reduced():
    aov = compare(vx.config.C1, [vx.Model.procedural(7, shell=False)], [0], w=128, h=128)
    assert (aov["object_id"] >= 0).mean() > 0.2
    aov = compare(vx.config.C4, [vx.Model.procedural(7, shell=True)], [0] * 64, w=192, h=108, t=1.3)
    assert (aov["object_id"] >= 0).sum() > 1000


def test_c2_animated_reduced():
    compare(vx.config.C2, [vx.Model.procedural(8, shell=True)], [0], w=160, h=90, t=2.2)
