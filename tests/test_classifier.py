"""CPU: the FP32 tie classifier (oracle/ref_harness.cpp: classify_rule) must not
accept wrong answers.

The FP32 kernel's hits are bit-exact vs the reference except for documented
slab-test ties, decided per pixel by geometric FP64 rules. These tests plant
wrong answers into a copy of the oracle's own per-pixel records -- another
voxel, instance, level, node or attribute index, a t past the stated
tolerance, a lost or invented hit -- and require the classifier to call them
bugs (or t-out-of-tolerance), except on the few pixels where a graze rule
legitimately accepts any answer (an instance's bounding sphere or root box is
grazed: the candidate sets themselves may differ there).
"""
import numpy as np
import pytest

import paper_1911_06001_b200 as vx
from oracle import ref

W, H = 320, 180
GRAZE = {ref.RULES[k] for k in (2, 3)}  # sphere / box graze rules


@pytest.fixture(scope="module")
def case():
    model = vx.Model.procedural(7, shell=True)
    om = ref.RefModel.from_bytes(model.serialize())
    sc = ref.RefScene(vx.config.C4, [om], 0, W, H)
    sc.evaluate(1.3)
    aov, _ = sc.dump()
    return sc, aov


def _rules(sc, o, g):
    return sc.classify_rules(o, g)


def _check_planted(sc, o, g, mask, allowed=("bug",)):
    r = _rules(sc, o, g)[mask]
    names = np.array([ref.RULES[int(v)] for v in r])
    assert not (names == "match").any(), "a planted error was classified as a match"
    ok = np.isin(names, list(allowed))
    graze = np.isin(names, list(GRAZE))
    assert (ok | graze).all(), ref.rule_histogram(r)
    assert ok.mean() >= 0.98, ref.rule_histogram(r)
    return ref.rule_histogram(r)


def test_identical_records_match(case):
    sc, o = case
    r = _rules(sc, o, o.copy())
    assert (r == 0).all()
    assert (o["object_id"] >= 0).sum() > 5000


def test_wrong_voxel_is_a_bug(case):
    sc, o = case
    hit = o["object_id"] >= 0
    g = o.copy()
    g["voxel"][hit, 0] = (g["voxel"][hit, 0] + 37) % 128  # depth 7: voxel coordinates < 128
    _check_planted(sc, o, g, hit)


def test_neighbour_voxel_off_the_ray_is_a_bug(case):
    sc, o = case
    hit = o["object_id"] >= 0
    g = o.copy()
    g["voxel"][hit, 1] = np.where(g["voxel"][hit, 1] >= 3, g["voxel"][hit, 1] - 3, g["voxel"][hit, 1] + 3)
    _check_planted(sc, o, g, hit)


def test_wrong_instance_is_a_bug(case):
    sc, o = case
    hit = o["object_id"] >= 0
    g = o.copy()
    g["object_id"][hit] = (g["object_id"][hit] + 29) % 64
    _check_planted(sc, o, g, hit)


def test_ancestor_or_descendant_level_is_a_bug(case):
    sc, o = case
    hit = o["object_id"] >= 0
    up = o.copy()  # the traversal stopping one level early: the parent cell
    up["level"][hit] -= 1
    up["voxel"][hit] >>= 1
    _check_planted(sc, o, up, hit)
    down = o.copy()  # one level too deep: a child cell of the oracle's voxel
    down["level"][hit] += 1
    down["voxel"][hit] <<= 1
    _check_planted(sc, o, down, hit)


def test_wrong_node_or_attribute_index_is_a_bug(case):
    sc, o = case
    hit = o["object_id"] >= 0
    g = o.copy()
    g["node_index"][hit] += 1
    r = _rules(sc, o, g)[hit]
    assert (r == ref.RULE_BUG).all()
    g = o.copy()
    g["attr_index"][hit] ^= 1
    r = _rules(sc, o, g)[hit]
    assert (r == ref.RULE_BUG).all()


def test_t_beyond_the_tolerance(case):
    sc, o = case
    hit = o["object_id"] >= 0
    g = o.copy()
    g["t"][hit] *= 1.0 + 2.0 ** -10  # past the 2^-12 cap of the grazing term
    r = _rules(sc, o, g)[hit]
    assert (r == ref.RULE_T_OUT).all(), ref.rule_histogram(r)
    g = o.copy()
    g["t"][hit] *= 1.0 + 2e-7  # FP32 rounding: inside the tolerance
    assert (_rules(sc, o, g)[hit] == 0).all()


def test_lost_hit_is_a_bug(case):
    sc, o = case
    hit = o["object_id"] >= 0
    g = o.copy()
    g["object_id"][hit] = -1
    _check_planted(sc, o, g, hit, allowed=("bug", "oracle_voxel_grazed", "miss_graze"))
    r = _rules(sc, o, g)[hit]
    assert (r == ref.RULE_BUG).mean() >= 0.98


def test_invented_hit_is_a_bug(case):
    sc, o = case
    miss = o["object_id"] < 0
    hits = np.flatnonzero((o["object_id"] >= 0).ravel())
    g = o.copy()
    flat = g.reshape(-1)
    src = flat[hits[np.arange(miss.sum()) % len(hits)]]
    flat[np.flatnonzero(miss.ravel())] = src  # another pixel's hit record on every miss pixel
    _check_planted(sc, o, g, miss)
