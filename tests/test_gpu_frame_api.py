"""GPU: render_frame semantics beyond the image — the hit buffer (HBO,
renderer.cpp:143-169,207-213,254-263), FrameStats, the multi-device screen
partition, and the error contract of the drop-in API."""
import ctypes as C

import numpy as np
import pytest

import paper_1911_06001_b200 as vx
from paper_1911_06001_b200 import _abi
from oracle import ref

pytestmark = pytest.mark.gpu


def hbo_pair(seed=414):
    models = [vx.Model.full_cube(), vx.Model.random(seed, 3, 0.3)]
    s = vx.Scene(vx.config.HBO, models)
    o = ref.RefScene(vx.config.HBO, [ref.RefModel.from_bytes(m.serialize()) for m in models])
    return s, o


def mutate(scene, frame, rng_t):
    """The reference HBO-transparency recipe (test_renderer.cpp:376-408)."""
    if frame % 3 == 1:
        oid, tf, _ = scene.get_object(2)
        tf[9:12] = [rng_t[0], 1.5 + rng_t[1], 1.0]
        scene.set_object(2, tf, True)
    if frame == 7:
        scene.set_object(0, scene.get_object(0)[1], True)
    if frame == 13:
        scene.set_camera_dirty(True)


@pytest.mark.parametrize("precision", [vx.VXA_FP64, vx.VXA_FP32])
def test_hbo_transparency_and_reference_stats(gpu, precision):
    s_hbo, o = hbo_pair()
    s_plain, _ = hbo_pair()
    hbo = vx.HitBuffer(96, 64)
    rhbo = ref.RefHitBuffer(96, 64)
    rng = np.random.default_rng(5)
    reused_total = 0
    for frame in range(25):
        jit = rng.uniform(-0.05, 0.05, 2)
        for sc in (s_hbo, s_plain, o):
            mutate(sc, frame, jit)
        a, _, sa = s_hbo.render(precision=precision, hbo=hbo)
        b, _, sb = s_plain.render(precision=precision)
        assert (a == b).all(), f"frame {frame}: hit buffer changed the image"
        assert sa["rays"] == 96 * 64
        reused_total += sa["pixels_reused"]
        if precision == vx.VXA_FP64:
            r_img, r_st = o.render(hbo=rhbo)
            assert (a == r_img).all(), f"frame {frame}: differs from the reference"
            for k in ("pixels_reused", "svo_traversals", "sphere_tests", "rays"):
                assert sa[k] == r_st[k], (frame, k, sa[k], r_st[k])
            # the GPU-resident HitBuffer, as the host sees it, equals the reference's records
            ours, theirs = hbo.records(), rhbo.records()
            for f in ("color", "normal", "t", "object_id", "kind"):
                assert (ours[f] == theirs[f]).all(), (frame, f)
            if frame in (9, 17):
                # a host write between frames reaches the next frame on both sides
                rec = theirs[20, 30].copy()
                rec["kind"], rec["object_id"] = 1, 1
                hbo.set_record(30, 20, rec)
                rhbo.set_record(30, 20, rec)
        for sc in (s_hbo, s_plain, o):
            sc.mark_clean()
    assert reused_total > 0


def test_hbo_dimension_mismatch_raises(gpu):
    s, _ = hbo_pair()
    with pytest.raises(vx.VoxanimError, match="hit buffer dimensions"):
        s.render(hbo=vx.HitBuffer(10, 10))


def test_screen_partition_composes_the_same_frame(gpu):
    """Ranks 0..world-1 rendering their super-tiles into one framebuffer (as the
    NVLink peer-store path does across GPUs) reproduce the single-device frame."""
    lib = vx.vxa()
    model = vx.Model.procedural(8, shell=True)
    s = vx.Scene(vx.config.C4, [model], 0, 1000, 600)
    s.evaluate(0.7)
    ctx = vx.context()
    f, inst, n = s.export()
    full = np.zeros((600, 1000, 3), np.uint8)
    assert lib.vxa_render(ctx, C.byref(f), inst, n, full.ctypes.data, None, None) == 0
    for world in (2, 3, 4, 8):
        for rank in range(world):
            f.tile_rank, f.tile_world = rank, world
            assert lib.vxa_submit(ctx, C.byref(f), inst, n) == 0, lib.vxa_last_error()
        part = np.zeros_like(full)
        assert lib.vxa_read_framebuffer(ctx, part.ctypes.data, 1000, 600) == 0
        assert (part == full).all(), f"world {world}"


def test_stats_and_launch_counts(gpu):
    model = vx.Model.procedural(8, shell=False)
    s = vx.Scene(vx.config.C1, [model])
    o = ref.RefScene(vx.config.C1, [ref.RefModel.from_bytes(model.serialize())])
    _, _, st = s.render(precision=vx.VXA_FP64)
    _, rst = o.render()
    for k in ("rays", "sphere_tests", "svo_traversals", "pixels_reused"):
        assert st[k] == rst[k], k
    assert st["kernel_launches"] == 1  # the frame kernel (it writes the RGB8 image itself)
    assert st["gpu_ms"] > 0


def test_invalid_arguments(gpu):
    lib = vx.vxa()
    ctx = vx.context()
    f = _abi.vxa_frame_desc()
    f.camera.width, f.camera.height, f.tile_world = 0, 10, 1
    assert lib.vxa_render(ctx, C.byref(f), None, 0, None, None, None) == _abi.VXA_ERR_INVALID
    f.camera.width, f.tile_world, f.tile_rank = 10, 2, 2
    assert lib.vxa_render(ctx, C.byref(f), None, 0, None, None, None) == _abi.VXA_ERR_INVALID
    # a model violating the SVO invariants (child_base <= parent) is refused
    bad = (C.c_uint8 * 12)(0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0)
    h = C.c_uint32()
    assert lib.vxa_upload_model(ctx, bad, 1, None, 0, 1, C.byref(h)) == _abi.VXA_ERR_MODEL
    # empty scene renders the background
    s = vx.Scene(vx.config.TWO_OBJECTS, [vx.Model.random(3, 2, 0.0)])
    img, _, st = s.render()
    assert (img == np.array([10, 20, 30], np.uint8)).all()


@pytest.mark.parametrize("precision", [vx.VXA_FP64, vx.VXA_FP32])
def test_device_hit_buffer_matches_host_hit_buffer(gpu, precision):
    """The device-resident HBO (vxa_hbo_create) follows the same reuse rule as the
    host HitBuffer: identical images and FrameStats over a mutating sequence, and
    (FP64) identical to the reference renderer with its HitBuffer."""
    lib = vx.vxa()
    ctx = vx.context()
    s_dev, o = hbo_pair(77)
    s_host, _ = hbo_pair(77)
    hbo_host = vx.HitBuffer(96, 64)
    rhbo = ref.RefHitBuffer(96, 64)
    handle = C.c_uint32()
    assert lib.vxa_hbo_create(ctx, 96, 64, C.byref(handle)) == 0
    rng = np.random.default_rng(9)
    for frame in range(20):
        jit = rng.uniform(-0.05, 0.05, 2)
        for sc in (s_dev, s_host, o):
            mutate(sc, frame, jit)
        f, inst, n = s_dev.export()
        f.precision = precision
        f.hbo_device = handle.value
        img = np.zeros((64, 96, 3), np.uint8)
        st = _abi.vxa_stats()
        assert lib.vxa_render(ctx, C.byref(f), inst, n, img.ctypes.data, None, C.byref(st)) == 0, \
            lib.vxa_last_error()
        b, _, sb = s_host.render(precision=precision, hbo=hbo_host)
        assert (img == b).all(), frame
        assert st.pixels_reused == sb["pixels_reused"] and st.svo_traversals == sb["svo_traversals"]
        if precision == vx.VXA_FP64:
            r_img, r_st = o.render(hbo=rhbo)
            assert (img == r_img).all()
            assert st.pixels_reused == r_st["pixels_reused"]
        for sc in (s_dev, s_host, o):
            sc.mark_clean()
    recs = (_abi.vxa_hit_record * (96 * 64))()
    assert lib.vxa_hbo_download(ctx, handle.value, recs) == 0
    assert any(r.kind != 0 for r in recs)
    assert lib.vxa_hbo_release(ctx, handle.value) == 0


def test_compact_fp32_hit_buffer_equals_full_records(gpu, monkeypatch):
    """FP32 frames keep device hit buffers in 16-byte records (normal rebuilt from
    the object's rotation and the stored local axis/sign). Over a mutating
    sequence that also switches to FP64 frames and back (format conversions both
    ways) and takes host writes, images and FrameStats equal those of the 48-byte
    path (VOXANIM_HBO_COMPACT=0), and so do the records the host sees (bit for bit
    until an FP64 frame's records pass through the compact format, which holds t
    and the normal to FP32 precision)."""
    runs = []
    for mode in ("1", "0"):
        monkeypatch.setenv("VOXANIM_HBO_COMPACT", mode)
        s, _ = hbo_pair(31)
        hbo = vx.HitBuffer(96, 64)
        rng = np.random.default_rng(3)
        out = []
        for frame in range(16):
            mutate(s, frame, rng.uniform(-0.05, 0.05, 2))
            prec = vx.VXA_FP64 if frame in (6, 7, 12) else vx.VXA_FP32
            img, _, st = s.render(precision=prec, hbo=hbo)
            recs = hbo.records()
            out.append((img, st["pixels_reused"], st["svo_traversals"], recs))
            if frame == 9:
                rec = recs[20, 30].copy()
                rec["kind"], rec["object_id"] = 1, 1
                hbo.set_record(30, 20, rec)
            s.mark_clean()
        runs.append(out)
    monkeypatch.delenv("VOXANIM_HBO_COMPACT")
    reused = 0
    for k, (a, b) in enumerate(zip(*runs)):
        assert (a[0] == b[0]).all(), k
        assert a[1] == b[1] and a[2] == b[2], k
        reused += a[1]
        for f in ("color", "object_id", "kind"):
            assert (a[3][f] == b[3][f]).all(), (k, f)
        if k < 6:  # FP32 frames only so far: the records agree bit for bit
            assert (a[3]["t"] == b[3]["t"]).all() and (a[3]["normal"] == b[3]["normal"]).all(), k
        else:
            # records an FP64 frame wrote and an FP32 frame kept hold t and the
            # normal to FP32 precision in the compact format
            assert np.allclose(a[3]["t"], b[3]["t"], rtol=1e-6, atol=0), k
            assert np.allclose(a[3]["normal"], b[3]["normal"], rtol=0, atol=1e-6), k
    assert reused > 0


@pytest.mark.parametrize("cfg,precision", [(vx.config.C4, vx.VXA_FP32), (vx.config.C2, vx.VXA_FP32),
                                           (vx.config.C2, vx.VXA_FP64)])
def test_banded_synchronous_readback(gpu, cfg, precision, monkeypatch):
    """A synchronous render of a large frame copies the RGB8 image in bands of
    super-tile rows, each started by a stream wait on the band's tile counter while
    the kernel renders the rest: the image equals the one copied after the kernel
    (VOXANIM_BANDED_READBACK=0), frame after frame, with and without the culling
    pre-pass's longest-first order (C4: 64 instances; C2: one)."""
    depth = 11 if cfg == vx.config.C4 else 10
    m = vx.Model.procedural(depth, shell=True)
    a, b = vx.Scene(cfg, [m]), vx.Scene(cfg, [m])
    for t in (0.2, 1.9, 3.4):
        a.evaluate(t)
        b.evaluate(t)
        monkeypatch.delenv("VOXANIM_BANDED_READBACK", raising=False)
        banded = a.render(precision=precision)[0]
        monkeypatch.setenv("VOXANIM_BANDED_READBACK", "0")
        plain = b.render(precision=precision)[0]
        monkeypatch.delenv("VOXANIM_BANDED_READBACK")
        assert (banded == plain).all(), t
        assert (banded != 0).any()


@pytest.mark.parametrize("cfg,precision,size", [(vx.config.C4, vx.VXA_FP32, None), (vx.config.C2, vx.VXA_FP32, None),
                                                (vx.config.C2, vx.VXA_FP64, None),
                                                (vx.config.C4, vx.VXA_FP32, (1008, 1040)),
                                                (vx.config.C4, vx.VXA_FP32, (1000, 1050))])
def test_direct_synchronous_readback(gpu, cfg, precision, size, monkeypatch):
    """A synchronous render into a page-locked (registered) host image: the warp
    finishing each super-tile stores its RGB8 rows into the image over PCIe during
    the frame. The image equals the one copied after the kernel
    (VOXANIM_DIRECT_READBACK=0 and VOXANIM_BANDED_READBACK=0), frame after frame;
    1008x1040 has partial super-tiles on the right and bottom edges, 1000x1050 rows
    that are not 16-byte multiples (the byte-wise copy)."""
    lib, ctx = vx.vxa(), vx.context()
    depth = 11 if cfg == vx.config.C4 else 10
    m = vx.Model.procedural(depth, shell=True)
    args = (0,) + size if size else ()
    a, b = vx.Scene(cfg, [m], *args), vx.Scene(cfg, [m], *args)
    img = np.zeros((a.height, a.width, 3), np.uint8)
    assert lib.vxa_host_register(ctx, img.ctypes.data, img.nbytes) == 0
    try:
        for t in (0.2, 1.9, 3.4):
            a.evaluate(t)
            b.evaluate(t)
            img[...] = 7
            monkeypatch.delenv("VOXANIM_DIRECT_READBACK", raising=False)
            a.render(precision=precision, rgb=img)
            monkeypatch.setenv("VOXANIM_DIRECT_READBACK", "0")
            monkeypatch.setenv("VOXANIM_BANDED_READBACK", "0")
            plain = b.render(precision=precision)[0]
            monkeypatch.delenv("VOXANIM_DIRECT_READBACK")
            monkeypatch.delenv("VOXANIM_BANDED_READBACK")
            assert (img == plain).all(), t
            assert (img != 0).any()
    finally:
        lib.vxa_host_unregister(ctx, img.ctypes.data)


def test_streaming_readback_matches_synchronous_frames(gpu):
    """vxa_submit_readback (frame k's D2H overlapping frame k+1) delivers the same
    images as synchronous render_frame calls."""
    lib = vx.vxa()
    ctx = vx.context()
    model = vx.Model.procedural(8, shell=True)
    s_stream = vx.Scene(vx.config.C4, [model], 0, 640, 360)
    s_sync = vx.Scene(vx.config.C4, [model], 0, 640, 360)
    vxl = vx.voxanim()
    bufs = [np.zeros((360, 640, 3), np.uint8) for _ in range(2)]
    for b in bufs:
        assert lib.vxa_host_register(ctx, b.ctypes.data, b.nbytes) == 0
    tickets, frames = [], []
    t = C.c_uint64()
    for k in range(6):
        assert vxl.vxn_scene_stream(s_stream._h, k / 30.0, vx.VXA_FP32, bufs[k % 2].ctypes.data, C.byref(t)) == 0
        tickets.append(t.value)
        s_sync.evaluate(k / 30.0)
        frames.append(s_sync.render(precision=vx.VXA_FP32)[0])
        s_sync.mark_clean()
        if k >= 1:
            assert lib.vxa_wait_readback(ctx, tickets[k - 1]) == 0
            assert (bufs[(k - 1) % 2] == frames[k - 1]).all(), k - 1
    assert lib.vxa_wait_readback(ctx, tickets[-1]) == 0
    assert (bufs[5 % 2] == frames[5]).all()
    for b in bufs:
        lib.vxa_host_unregister(ctx, b.ctypes.data)


def test_concurrent_render_calls_from_host_threads(gpu):
    """render_frame from several host threads at once (the reference's renderer
    has no shared state, so callers may do this): every call serialises on the
    process-wide context and returns exactly its sequential frame."""
    import threading

    models = [vx.Model.procedural(6, shell=True), vx.Model.random(7, 4, 0.3)]
    scenes = [vx.Scene(cfg, models, 3, 160, 96) for cfg in (vx.config.RANDOM, vx.config.HBO, vx.config.C1,
                                                             vx.config.MANY)]
    times = [0.0, 0.4, 0.0, 0.0]
    expected = []
    for sc, t in zip(scenes, times):
        sc.evaluate(t)
        expected.append([sc.render(precision=p)[0] for p in (vx.VXA_FP32, vx.VXA_FP64)])
    errors = []

    def worker(k):
        try:
            for _ in range(6):
                for j, p in enumerate((vx.VXA_FP32, vx.VXA_FP64)):
                    img = scenes[k].render(precision=p)[0]
                    if not (img == expected[k][j]).all():
                        errors.append((k, p))
        except Exception as e:  # surfaced below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(len(scenes))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors


def test_c_abi_misuse_is_reported_not_fatal(gpu):
    """Unknown handles, double releases, unknown readback tickets and null
    arguments return status codes; an instance whose model handle is unknown is
    skipped like a reference object without a model (renderer.cpp:74-76)."""
    lib = vx.vxa()
    ctx = vx.context()
    inv = _abi.VXA_ERR_INVALID
    assert lib.vxa_release_model(ctx, 987654) == inv
    assert lib.vxa_hbo_release(ctx, 987654) == inv
    assert lib.vxa_model_info(ctx, 987654, None, None) == inv
    assert lib.vxa_wait_readback(ctx, 1 << 40) == inv
    assert lib.vxa_build_model(ctx, None, 3, 0, 0, None, None, None) == inv
    h = C.c_uint32()
    m = vx.Model.random(5, 3, 0.5).serialize()
    assert lib.vxa_upload_svo(ctx, m, len(m), C.byref(h), None) == 0
    assert lib.vxa_release_model(ctx, h.value) == 0
    assert lib.vxa_release_model(ctx, h.value) == inv  # double release
    # an instance pointing at no model: skipped, the frame equals the frame without it
    s = vx.Scene(vx.config.TWO_OBJECTS, [vx.Model.random(4, 3, 0.4)])
    f, inst, n = s.export()
    with_ghost = np.zeros((s.height, s.width, 3), np.uint8)
    inst[0].model = 987654
    assert lib.vxa_render(ctx, C.byref(f), inst, n, with_ghost.ctypes.data, None, None) == 0
    without = np.zeros_like(with_ghost)
    assert lib.vxa_render(ctx, C.byref(f), C.byref(inst[1]), 1, without.ctypes.data, None, None) == 0
    assert (with_ghost == without).all()


def test_back_to_back_frames_with_growing_instance_tables(gpu):
    """Frames submitted without waiting, alternating a 64-instance and a 700-instance
    scene on one context: the double-buffered device instance tables grow while
    earlier frames are in flight, and every frame equals its synchronous render."""
    lib = vx.vxa()
    ctx = vx.context()
    vxl = vx.voxanim()
    model = vx.Model.procedural(6, shell=True)
    small = vx.Scene(vx.config.C4, [model], 0, 320, 180)
    big = vx.Scene(vx.config.CROWD, [model], 700, 320, 180)
    bufs = [np.zeros((180, 320, 3), np.uint8) for _ in range(2)]
    for b in bufs:
        assert lib.vxa_host_register(ctx, b.ctypes.data, b.nbytes) == 0
    t = C.c_uint64()
    tickets, scenes = [], []
    for k in range(8):
        sc = big if k % 2 else small
        assert vxl.vxn_scene_stream(sc._h, k / 30.0, vx.VXA_FP32, bufs[k % 2].ctypes.data, C.byref(t)) == 0
        tickets.append(t.value)
        scenes.append(sc)
        if k >= 1:
            assert lib.vxa_wait_readback(ctx, tickets[k - 1]) == 0
            got = bufs[(k - 1) % 2].copy()
            ref_sc = scenes[k - 1]
            # the synchronous frame of the same scene and time, rendered after the stream caught up
            assert lib.vxa_wait_readback(ctx, tickets[k]) == 0
            ref_sc.evaluate((k - 1) / 30.0)
            want = ref_sc.render(precision=vx.VXA_FP32)[0]
            assert (got == want).all(), k - 1
    for b in bufs:
        lib.vxa_host_unregister(ctx, b.ctypes.data)


def test_stream_delay_holds_the_stream(gpu):
    """vxa_stream_delay (bench head start) keeps the context stream busy for the
    requested time and nothing else."""
    lib = vx.vxa()
    ctx = vx.context()
    ms = C.c_double()
    assert lib.vxa_timer_begin(ctx) == 0
    assert lib.vxa_stream_delay(ctx, 300) == 0
    assert lib.vxa_timer_end(ctx, C.byref(ms)) == 0
    assert 0.29 <= ms.value < 5.0, ms.value


@pytest.mark.parametrize("staged,spares", [("1", "1"), ("1", "0"), ("0", "0")])
def test_drop_in_render_frame_image(gpu, staged, spares, monkeypatch):
    """The drop-in voxanim::render_frame returns its Image by value; a large frame is
    rendered into a page-locked staging image (direct readback) while a worker takes
    the Image (a ready zero-filled one, or VOXANIM_IMAGE_SPARES=0 built then), then
    copied in parallel (VOXANIM_IMAGE_STAGING=0: straight into the Image). All give
    the render_frame_into image, frame after frame, also when the frame size changes."""
    vxl = vx.voxanim()
    monkeypatch.setenv("VOXANIM_IMAGE_STAGING", staged)
    monkeypatch.setenv("VOXANIM_IMAGE_SPARES", spares)
    m = vx.Model.procedural(10, shell=True)
    a, b = vx.Scene(vx.config.C4, [m], 0, 1920, 1080), vx.Scene(vx.config.C4, [m], 0, 1920, 1080)
    last = np.zeros((1080, 1920, 3), np.uint8)
    ms = C.c_double()
    for t in (0.3, 2.1):
        assert vxl.vxn_scene_render_image(a._h, t, 3, C.byref(ms), last.ctypes.data) == 0
        b.evaluate(t + 2 / 30.0)
        want = b.render()[0]
        assert (last == want).all(), t
        assert ms.value > 0.0
    # another frame size: the ready images of the old size are not used
    a2, b2 = vx.Scene(vx.config.C4, [m], 0, 1280, 1024), vx.Scene(vx.config.C4, [m], 0, 1280, 1024)
    last2 = np.zeros((1024, 1280, 3), np.uint8)
    assert vxl.vxn_scene_render_image(a2._h, 1.0, 2, C.byref(ms), last2.ctypes.data) == 0
    b2.evaluate(1.0 + 1 / 30.0)
    assert (last2 == b2.render()[0]).all()
