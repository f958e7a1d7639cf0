"""GPU: the device SVO builder (vxa_build_model, csrc/cuda/build.cu) replacing
the reference's build_from_grid (proj/src/svo.cpp:52-132). Parity bar: the
serialized model (every 12-byte node record and every attribute) identical byte
for byte to the reference build on the same VoxelGrid, for random grids, the
reference primitives, the edge cases and every colour mode; at depth 10 (where
the reference needs ~48 s / 15 GB) against the product's host builder, itself
pinned to the reference by tests/test_grid_build.py and test_builder.py."""
import ctypes as C

import numpy as np
import pytest

import paper_1911_06001_b200 as vx
from oracle import ref
from test_grid_build import MODES, edge_grids, random_grid

pytestmark = pytest.mark.gpu


def device_bytes(words, depth, mode=0, rgba=0xFFC8C8C8):
    return vx.Model.from_grid(words, depth, mode, rgba, device=True).serialize()


@pytest.mark.parametrize("mode,rgba", MODES)
def test_random_grids_bit_exact(gpu, mode, rgba):
    for seed, depth, fill in [(1, 2, 0.5), (2, 4, 0.1), (3, 5, 0.02), (4, 6, 0.3), (5, 3, 0.9), (6, 7, 0.01),
                              (7, 8, 0.001)]:
        w = random_grid(seed, depth, fill)
        assert device_bytes(w, depth, mode, rgba) == ref.RefModel.from_grid(w, depth, mode, rgba).serialize(), \
            (seed, depth, fill, mode)


def test_edge_grids_bit_exact(gpu):
    for name, words, depth in edge_grids():
        assert device_bytes(words, depth) == ref.RefModel.from_grid(words, depth).serialize(), name


@pytest.mark.parametrize("kind", sorted(vx.PRIMITIVES))
def test_primitives_bit_exact(gpu, kind):
    for depth in (1, 3, 5, 8) if kind != "menger" else (1, 3, 5):
        words, gd = vx.grid_primitive(kind, depth)
        assert device_bytes(words, gd, 1) == ref.RefModel.from_grid(words, gd, 1).serialize(), (kind, depth)


def test_reference_c1_model(gpu):
    """C1's model: the reference's gen_primitive(Sphere, 8) -> build_from_grid."""
    words, gd = vx.grid_primitive("sphere", 8)
    dev = vx.Model.from_grid(words, gd, device=True)
    assert dev.info() == {"depth": 8, "nodes": 1284089, "attributes": 8783848}
    assert dev.serialize() == ref.RefModel.dense_sphere(8).serialize()


def test_depth10_matches_host_builder(gpu):
    words, gd = vx.grid_primitive("sphere", 10)
    dev = vx.Model.from_grid(words, gd, 0, device=True)
    host = vx.Model.from_grid(words, gd, 0, device=False)
    assert dev.info() == host.info()
    assert dev.serialize() == host.serialize()
    assert dev.violations() == 0


def test_built_model_renders_like_uploaded(gpu):
    """A device-built model is registered in the model cache at build time; the
    frame rendered from it equals the frame of the same model uploaded from
    host records (and, FP64, the reference frame)."""
    words, gd = vx.grid_primitive("sphere", 6)
    built = vx.Model.from_grid(words, gd, device=True)
    uploaded = vx.Model.from_bytes(built.serialize())
    a = vx.Scene(vx.config.C1, [built]).render(precision=vx.VXA_FP64)[0]
    b = vx.Scene(vx.config.C1, [uploaded]).render(precision=vx.VXA_FP64)[0]
    o = ref.RefScene(vx.config.C1, [ref.RefModel.from_grid(words, gd)]).render()[0]
    assert (a == b).all() and (a == o).all()


@pytest.mark.parametrize("prim,depth", [("sphere", 7), ("box_shell", 6), ("menger", 6)])
def test_built_model_content_bound_renders_like_uploaded_fp32(gpu, prim, depth):
    """The FP32 kernel skips traversals of rays missing the model's content
    sphere. Device-built models get it from the builder's leaf extent reduction,
    uploaded ones from the host walk: both conservative, so the FP32 frames of the
    same model agree pixel for pixel, in the C1 view and the 64-instance C4 layout."""
    words, gd = vx.grid_primitive(prim, depth)
    built = vx.Model.from_grid(words, gd, device=True)
    uploaded = vx.Model.from_bytes(built.serialize())
    for cfg, w, h in ((vx.config.C1, 0, 0), (vx.config.C4, 480, 270)):
        sa = vx.Scene(cfg, [built], 0, w, h)
        sb = vx.Scene(cfg, [uploaded], 0, w, h)
        sa.evaluate(0.7)
        sb.evaluate(0.7)
        a = sa.render(precision=vx.VXA_FP32)[0]
        b = sb.render(precision=vx.VXA_FP32)[0]
        assert (a == b).all(), (prim, cfg)


@pytest.mark.parametrize("prim,depth", [("sphere", 7), ("box_shell", 6), ("menger", 6), ("full", 5)])
def test_built_model_content_bound_never_changes_a_frame(gpu, prim, depth, monkeypatch):
    """The content bound is only a skip: FP32 frames of device-built models with
    the content-sphere test on and off (VOXANIM_CONTENT_BOUND=off) agree pixel for
    pixel -- incl. models whose leaves reach the cube's corners (box shell, full
    cube: the bound must not cut them) -- in the C1 view and the C4 layout."""
    if prim == "full":
        n = 1 << depth
        words = np.full((n ** 3 + 63) // 64, np.iinfo(np.uint64).max, np.uint64)
        gd = depth
    else:
        words, gd = vx.grid_primitive(prim, depth)
    built = vx.Model.from_grid(words, gd, device=True)
    for cfg, w, h in ((vx.config.C1, 0, 0), (vx.config.C4, 480, 270)):
        sc = vx.Scene(cfg, [built], 0, w, h)
        sc.evaluate(0.7)
        monkeypatch.delenv("VOXANIM_CONTENT_BOUND", raising=False)
        on = sc.render(precision=vx.VXA_FP32)[0]
        monkeypatch.setenv("VOXANIM_CONTENT_BOUND", "off")
        off = sc.render(precision=vx.VXA_FP32)[0]
        monkeypatch.delenv("VOXANIM_CONTENT_BOUND")
        assert (on == off).all(), (prim, cfg)
        assert (on != 0).any()


def test_c_abi_build_download_and_errors(gpu):
    lib = vx.vxa()
    ctx = vx.context()
    w = random_grid(11, 5, 0.2)
    h, nn, na = C.c_uint32(), C.c_uint64(), C.c_uint64()
    assert lib.vxa_build_model(ctx, w.ctypes.data, 5, 0, 0, C.byref(h), C.byref(nn), C.byref(na)) == 0
    nodes = np.zeros(nn.value * 12, np.uint8)
    attrs = np.zeros(na.value, np.uint32)
    assert lib.vxa_model_download(ctx, h.value, nodes.ctypes.data, nn.value, attrs.ctypes.data, na.value) == 0
    r = ref.RefModel.from_grid(w, 5).serialize()
    assert nodes.tobytes() == r[20:20 + 12 * nn.value]
    assert attrs.tobytes() == r[20 + 12 * nn.value:]
    fmt = C.c_uint32()
    assert lib.vxa_model_info(ctx, h.value, None, C.byref(fmt)) == 0 and fmt.value == 1  # compact words
    assert lib.vxa_model_download(ctx, h.value, nodes.ctypes.data, nn.value - 1, None, 0) == _abi_invalid()
    assert lib.vxa_release_model(ctx, h.value) == 0
    assert lib.vxa_build_model(ctx, w.ctypes.data, 11, 0, 0, C.byref(h), None, None) == _abi_invalid()
    assert lib.vxa_build_model(ctx, w.ctypes.data, 5, 3, 0, C.byref(h), None, None) == _abi_invalid()
    with pytest.raises(vx.VoxanimError):
        vx.Model.from_grid(np.zeros(8, np.uint64), 3, color_mode=5, device=True)


def _abi_invalid():
    from paper_1911_06001_b200 import _abi
    return _abi.VXA_ERR_INVALID


def _corruptions(good: bytes):
    """One stream per SvoFormatErrorCode class (test_svo.cpp's corruption cases)."""
    import struct
    n_nodes = struct.unpack_from("<I", good, 12)[0]
    yield "short header", good[:19]
    yield "bad magic", b"XVOA" + good[4:]
    yield "bad version", good[:4] + struct.pack("<I", 2) + good[8:]
    yield "depth 0", good[:8] + struct.pack("<I", 0) + good[12:]
    yield "depth 17", good[:8] + struct.pack("<I", 17) + good[12:]
    yield "no nodes", good[:12] + struct.pack("<I", 0) + good[16:]
    yield "truncated payload", good[:-1]
    yield "trailing data", good + b"\0"
    b = bytearray(good)
    struct.pack_into("<I", b, 20, n_nodes)  # root child_base past the end
    yield "child out of range", bytes(b)
    last = 20 + 12 * (n_nodes - 1)  # a last-level node: attr_base past the end
    b = bytearray(good)
    struct.pack_into("<I", b, last + 4, 1 << 30)
    yield "attr out of range", bytes(b)


def test_upload_svo_stream(gpu):
    """vxa_upload_svo: a well-formed stream renders like the uploaded SvoModel;
    every corruption class fails with the reference deserialize()'s message."""
    lib = vx.vxa()
    ctx = vx.context()
    model = vx.Model.random(21, 4, 0.2)
    good = model.serialize()
    h, code = C.c_uint32(), C.c_int32()
    assert lib.vxa_upload_svo(ctx, good, len(good), C.byref(h), C.byref(code)) == 0 and code.value == -1
    nodes = np.zeros(len(good), np.uint8)
    n_nodes = int(np.frombuffer(good[12:16], np.uint32)[0])
    assert lib.vxa_model_download(ctx, h.value, nodes.ctypes.data, n_nodes, None, 0) == 0
    assert nodes[:12 * n_nodes].tobytes() == good[20:20 + 12 * n_nodes]
    lib.vxa_release_model(ctx, h.value)
    expected_code = {"short header": 3, "bad magic": 0, "bad version": 1, "depth 0": 2, "depth 17": 2,
                     "no nodes": 2, "truncated payload": 3, "trailing data": 4, "child out of range": 5,
                     "attr out of range": 6}
    for name, data in _corruptions(good):
        with pytest.raises(RuntimeError) as ref_err:
            ref.RefModel.from_bytes(data)
        rc = lib.vxa_upload_svo(ctx, data, len(data), C.byref(h), C.byref(code))
        assert rc == 2, name  # VXA_ERR_MODEL
        assert code.value == expected_code[name], name
        assert lib.vxa_last_error().decode() == str(ref_err.value), name
