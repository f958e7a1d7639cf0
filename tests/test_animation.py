"""CPU: the per-frame host update is bit-identical to the reference.

evaluate_animation / evaluate_track (reference scene.cpp:345-385) produce the
RigidTransforms the GPU frame consumes; the benchmark scenes (bench_scenes.cpp)
are compiled against both implementations, so every transform component and
every dirty flag must be equal bit for bit over whole sequences.
"""
import pytest

import paper_1911_06001_b200 as vx
from oracle import ref


def scenes(cfg, model, w=64, h=36):
    return vx.Scene(cfg, [model], 0, w, h), ref.RefScene(cfg, [ref.RefModel.from_bytes(model.serialize())], 0, w, h)


@pytest.mark.parametrize("cfg", [vx.config.C2, vx.config.C4])
def test_sequence_transforms_bit_identical(cfg):
    model = vx.Model.procedural(3, shell=True)
    s, o = scenes(cfg, model)
    n = s.object_count()
    for frame in list(range(0, 130)) + [200, 500]:
        t = frame / 30.0
        s.evaluate(t)
        o.evaluate(t)
        for i in range(n):
            assert s.get_object(i) == o.get_object(i), (frame, i)
        s.mark_clean()
        o.mark_clean()


def test_static_scene_stays_clean():
    model = vx.Model.procedural(3, shell=True)
    s, o = scenes(vx.config.C3, model)
    for t in (0.0, 1.0, 2.5):
        s.evaluate(t)
        o.evaluate(t)
        assert s.get_object(0) == o.get_object(0)
        assert s.get_object(0)[2] is False


def test_negative_time_is_rejected():
    model = vx.Model.procedural(2, shell=True)
    s, o = scenes(vx.config.C2, model)
    with pytest.raises(vx.VoxanimError):
        s.evaluate(-0.5)
    with pytest.raises(RuntimeError):
        o.evaluate(-0.5)
