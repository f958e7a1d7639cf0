"""voxanim-b200: B200-native animated-SVO ray casting behind the voxanim C++ API.

The product is native: lib/libvxa.so (CUDA kernels for sm_100a + the C ABI of
include/vxa.h) and lib/libvoxanim.so (the drop-in voxanim:: C++ API of the
reference, proj/include/voxanim/*.hpp, whose render_frame/traverse call the
C ABI). This module is a thin ctypes veneer over include/voxanim_capi.h for
tests and bench.py; it performs no computation itself.
"""
from __future__ import annotations

import ctypes as C

from . import _abi
from ._abi import (AOV_DTYPE, HBO_DTYPE, RAY_DTYPE, TRAV_DTYPE, VXA_FP32, VXA_FP64, vxa_frame_desc, vxa_instance,
                   vxa_stats)

__all__ = ["Model", "Scene", "HitBuffer", "traverse", "vxa", "voxanim", "VoxanimError", "VXA_FP32", "VXA_FP64",
           "AOV_DTYPE", "RAY_DTYPE", "TRAV_DTYPE", "config"]

_VXA = None
_VX = None


class VoxanimError(RuntimeError):
    pass


def vxa() -> C.CDLL:
    """libvxa.so (C ABI of the CUDA layer)."""
    global _VXA
    if _VXA is None:
        _VXA = _abi.load_vxa()
    return _VXA


def voxanim() -> C.CDLL:
    """libvoxanim.so (voxanim:: C++ API + flat C binding)."""
    global _VX
    if _VX is None:
        vxa()
        _VX = _abi.load_voxanim()
    return _VX


def _err() -> str:
    return voxanim().vxn_last_error().decode()


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise VoxanimError(f"{what}: {_err()}")


class config:  # bench_scenes.hpp
    C1 = 1
    C2 = 2
    C3 = 3
    C4 = 4
    RANDOM = 5
    SORTED_TRACING = 6
    TWO_OBJECTS = 7
    HBO = 8
    AXIS_ALIGNED = 9
    MANY = 10
    CROWD = 11     # seed = instance count (0: 4096)
    STACKED = 12


class Model:
    """shared_ptr<const voxanim::SvoModel>."""

    def __init__(self, handle):
        if not handle:
            raise VoxanimError(_err())
        self._h = C.c_void_p(handle)

    @classmethod
    def procedural(cls, depth: int, shell: bool = True) -> "Model":
        return cls(voxanim().vxn_model_procedural(1 if shell else 0, depth))

    @classmethod
    def dense_sphere(cls, depth: int) -> "Model":
        return cls(voxanim().vxn_model_dense_sphere(depth))

    @classmethod
    def random(cls, seed: int, depth: int, fill: float) -> "Model":
        return cls(voxanim().vxn_model_random(seed, depth, fill))

    @classmethod
    def full_cube(cls) -> "Model":
        return cls(voxanim().vxn_model_full_cube())

    @classmethod
    def from_grid(cls, words, depth: int, color_mode: int = 0, color_rgba: int = 0xFFC8C8C8,
                  device: bool = True) -> "Model":
        """build_from_grid of a VoxelGrid bitset (uint64 words, x-major); on the
        GPU (vxa_build_model) unless device=False."""
        import numpy as np
        w = np.ascontiguousarray(words, dtype=np.uint64)
        n = 1 << depth
        if w.size != (n ** 3 + 63) // 64:
            raise VoxanimError(f"grid has {w.size} words, expected {(n ** 3 + 63) // 64}")
        return cls(voxanim().vxn_model_from_grid(w.ctypes.data, depth, color_mode, color_rgba, 1 if device else 0))

    @classmethod
    def from_bytes(cls, data: bytes) -> "Model":
        buf = C.create_string_buffer(data, len(data))
        return cls(voxanim().vxn_model_deserialize(buf, len(data)))

    def save(self, path: str) -> None:
        """voxanim::save_svo."""
        _check(voxanim().vxn_model_save(self._h, str(path).encode()), "save_svo")

    def serialize(self) -> bytes:
        n = voxanim().vxn_model_serialize(self._h, None, 0)
        if n < 0:
            raise VoxanimError(_err())
        buf = C.create_string_buffer(n)
        voxanim().vxn_model_serialize(self._h, buf, n)
        return buf.raw

    def info(self) -> dict:
        d, n, a = C.c_uint32(), C.c_uint64(), C.c_uint64()
        voxanim().vxn_model_info(self._h, C.byref(d), C.byref(n), C.byref(a))
        return {"depth": d.value, "nodes": n.value, "attributes": a.value}

    def violations(self) -> int:
        return voxanim().vxn_model_validate(self._h)

    def __del__(self):
        if getattr(self, "_h", None) and _VX is not None:
            _VX.vxn_model_free(self._h)
            self._h = None


PRIMITIVES = {"sphere": 0, "box_shell": 1, "menger": 2, "checker": 3}


def grid_primitive(kind: str, depth: int):
    """gen_primitive(kind, depth) as (VoxelGrid bitset as numpy uint64 words,
    grid depth = log2 of its resolution)."""
    import numpy as np
    gd = C.c_uint32()
    n = voxanim().vxn_grid_primitive(PRIMITIVES[kind], depth, None, 0, C.byref(gd))
    if n < 0:
        raise VoxanimError(_err())
    out = np.zeros(n, np.uint64)
    if voxanim().vxn_grid_primitive(PRIMITIVES[kind], depth, out.ctypes.data, out.size, C.byref(gd)) < 0:
        raise VoxanimError(_err())
    return out, gd.value


class HitBuffer:
    def __init__(self, width: int, height: int):
        h = voxanim().vxn_hbo_create(width, height)
        if not h:
            raise VoxanimError(_err())
        self._h = C.c_void_p(h)
        self.width, self.height = width, height

    def records(self):
        """The records as the host sees them (HitBuffer::data): numpy HBO_DTYPE, height x width."""
        import numpy as np
        out = np.zeros((self.height, self.width), HBO_DTYPE)
        _check(voxanim().vxn_hbo_records(self._h, out.ctypes.data), "hbo_records")
        return out

    def set_record(self, x: int, y: int, rec) -> None:
        """HitBuffer::at(x, y) = rec (a HBO_DTYPE scalar)."""
        import numpy as np
        r = np.array(rec, HBO_DTYPE)
        _check(voxanim().vxn_hbo_set_record(self._h, x, y, r.ctypes.data), "hbo_set_record")

    def __del__(self):
        if getattr(self, "_h", None) and _VX is not None:
            _VX.vxn_hbo_free(self._h)
            self._h = None


class Scene:
    """voxanim::Scene built from a bench configuration (bench_scenes.hpp)."""

    def __init__(self, cfg: int, models, seed: int = 0, width: int = 0, height: int = 0):
        self.models = list(models)
        arr = (C.c_void_p * len(self.models))(*[m._h for m in self.models])
        h = voxanim().vxn_scene_config(cfg, arr, len(self.models), seed, width, height)
        if not h:
            raise VoxanimError(_err())
        self._h = C.c_void_p(h)
        f = vxa_frame_desc()
        _check(voxanim().vxn_scene_export(self._h, C.byref(f), None, 0, None), "export")
        self.width, self.height = f.camera.width, f.camera.height

    @classmethod
    def load(cls, path: str, width: int = 640, height: int = 480) -> "Scene":
        """voxanim::load_scene_file(path), camera resolution width x height."""
        h = voxanim().vxn_scene_load(str(path).encode(), width, height)
        if not h:
            raise VoxanimError(_err())
        self = cls.__new__(cls)
        self.models = []
        self._h = C.c_void_p(h)
        self.width, self.height = width, height
        return self

    def evaluate(self, t: float) -> None:
        _check(voxanim().vxn_scene_evaluate(self._h, t), "evaluate_animation")

    def mark_clean(self) -> None:
        voxanim().vxn_scene_mark_clean(self._h)

    def set_camera(self, position, look_at, up=(0.0, 1.0, 0.0), fov_deg=60.0, width=None, height=None) -> None:
        """camera = make_look_at_camera(...) (dirty); the resolution is kept unless given."""
        w, h = width or self.width, height or self.height
        P3 = C.c_double * 3
        _check(voxanim().vxn_scene_set_camera(self._h, P3(*position), P3(*look_at), P3(*up), float(fov_deg), w, h),
               "set_camera")
        self.width, self.height = w, h

    def set_camera_dirty(self, dirty: bool) -> None:
        voxanim().vxn_scene_set_camera_dirty(self._h, 1 if dirty else 0)

    def object_count(self) -> int:
        return voxanim().vxn_scene_object_count(self._h)

    def get_object(self, i: int):
        oid, tf, dirty = C.c_int32(), (C.c_double * 15)(), C.c_int()
        _check(voxanim().vxn_scene_get_object(self._h, i, C.byref(oid), tf, C.byref(dirty)), "get_object")
        return oid.value, list(tf), bool(dirty.value)

    def set_object(self, i: int, transform15, dirty: bool) -> None:
        tf = (C.c_double * 15)(*transform15)
        _check(voxanim().vxn_scene_set_object(self._h, i, tf, 1 if dirty else 0), "set_object")

    def frame_desc(self) -> vxa_frame_desc:
        """Camera + background as a vxa_frame_desc (host only, no device needed)."""
        f = vxa_frame_desc()
        _check(voxanim().vxn_scene_export(self._h, C.byref(f), None, 0, None), "export")
        return f

    def export(self):
        """(vxa_frame_desc, vxa_instance array) — the C-ABI view of the scene."""
        n = self.object_count()
        f = vxa_frame_desc()
        inst = (vxa_instance * max(n, 1))()
        cnt = C.c_uint32()
        _check(voxanim().vxn_scene_export(self._h, C.byref(f), inst, n, C.byref(cnt)), "export")
        return f, inst, cnt.value

    def render(self, culling=True, sorting=True, precision=None, hbo: HitBuffer | None = None, rgb=True,
               aov=False):
        """voxanim::render_frame on the GPU. Returns (rgb HxWx3 uint8 | None, aov | None, stats dict)."""
        import numpy as np

        W, H = self.width, self.height
        if isinstance(rgb, np.ndarray):
            assert rgb.shape == (H, W, 3) and rgb.dtype == np.uint8 and rgb.flags.c_contiguous
            img = rgb
        else:
            img = np.empty((H, W, 3), np.uint8) if rgb else None
        rgb = img is not None
        aovs = np.zeros((H, W), AOV_DTYPE) if aov else None
        fs = (C.c_uint64 * 4)()
        ms = C.c_double()
        ds = vxa_stats()
        prec = -1 if precision is None else int(precision)
        rc = voxanim().vxn_render(self._h, int(culling), int(sorting), prec, hbo._h if hbo else None,
                                  img.ctypes.data if rgb else None, aovs.ctypes.data if aov else None, fs,
                                  C.byref(ms), C.byref(ds))
        _check(rc, "render_frame")
        stats = {"rays": fs[0], "sphere_tests": fs[1], "svo_traversals": fs[2], "pixels_reused": fs[3],
                 "render_ms": ms.value, "node_fetches": ds.node_fetches, "leaf_hits": ds.leaf_hits,
                 "gpu_ms": ds.gpu_ms, "kernel_launches": ds.kernel_launches}
        return img, aovs, stats

    def __del__(self):
        if getattr(self, "_h", None) and _VX is not None:
            _VX.vxn_scene_free(self._h)
            self._h = None


def traverse(model: Model, rays):
    """voxanim::traverse for a RAY_DTYPE array (GPU, FP64 parity kernel)."""
    import numpy as np

    rays = np.ascontiguousarray(rays, dtype=RAY_DTYPE)
    out = np.zeros(len(rays), TRAV_DTYPE)
    _check(voxanim().vxn_traverse(model._h, rays.ctypes.data, len(rays), out.ctypes.data), "traverse")
    return out


def context():
    """The process-wide vxa_ctx* used by render_frame (for timers / L2 flush)."""
    h = voxanim().vxn_context()
    if not h:
        raise VoxanimError(_err())
    return C.c_void_p(h)
