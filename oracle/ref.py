"""TEST INFRASTRUCTURE — ctypes binding of the reference oracle (oracle/_ref/libvoxanim_ref.so).

The library is the reference CPU implementation (proj/src/*.cpp, compiled in
place by oracle/Makefile) plus oracle/ref_harness.cpp glue. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libvoxanim_ref.so")

AOV_DTYPE = np.dtype(
    [("t", "<f8"), ("object_id", "<i4"), ("node_index", "<u4"), ("attr_index", "<u4"), ("voxel", "<u4", (3,)),
     ("level", "u1"), ("kind", "u1"), ("entry_axis", "u1"), ("pad0", "u1"), ("traversals", "<u4"),
     ("node_fetches", "<u4"), ("pad1", "<u4")]
)
RAY_DTYPE = np.dtype([("origin", "<f8", (3,)), ("direction", "<f8", (3,)), ("half_extent", "<f8", (3,))])
TRAV_DTYPE = np.dtype(
    [("t_hit", "<f8"), ("t_enter", "<f8"), ("t_exit", "<f8"), ("normal_local", "<f8", (3,)),
     ("attribute", "u1", (4,)), ("attr_index", "<u4"), ("node_index", "<u4"), ("leaf_path", "u1", (16,)),
     ("path_len", "u1"), ("hit", "u1"), ("pad", "<u2"), ("node_fetches", "<u4"), ("log_count", "<u4"),
     ("log_total", "<u4")],
    align=True,
)

# default resolutions of the bench_scenes.hpp configurations
CONFIG_SIZES = {1: (512, 512), 2: (1920, 1080), 3: (1920, 1080), 4: (3840, 2160), 5: (160, 120), 6: (64, 48),
                7: (96, 64), 8: (96, 64), 9: (101, 101), 10: (320, 180), 11: (3840, 2160), 12: (160, 120)}

# classify() codes
MATCH, TIE, BUG, T_OUT_OF_TOL = 0, 1, 2, 3
# classify_rules() codes: 0 match, 1..10 the tie rules (oracle/ref_harness.cpp: Rule), 100 bug, 101 t out of tolerance
RULES = {0: "match", 1: "entry_face", 2: "sphere_graze", 3: "box_graze", 4: "zero_dir_face", 5: "oracle_voxel_grazed",
         6: "gpu_voxel_near_miss", 7: "behind_origin", 8: "same_entry_t", 9: "instance_tie", 10: "miss_graze",
         100: "bug", 101: "t_out_of_tolerance"}
RULE_BUG, RULE_T_OUT = 100, 101

_LIB = None
P = C.c_void_p


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not available():
            raise RuntimeError(f"oracle library {LIB_PATH} missing: run `make -C oracle` (needs /root/reference)")
        L = C.CDLL(LIB_PATH)
        i, u32, u64, d = C.c_int, C.c_uint32, C.c_uint64, C.c_double
        sig = {
            "vref_last_error": (C.c_char_p,),
            "vref_model_deserialize": (P, P, C.c_size_t),
            "vref_model_dense_sphere": (P, u32),
            "vref_model_load": (P, C.c_char_p),
            "vref_model_shell_grid": (P, u32),
            "vref_model_random": (P, u64, u32, d),
            "vref_model_from_grid": (P, P, u32, u32, u32),
            "vref_model_serialize": (C.c_int64, P, P, C.c_size_t),
            "vref_model_validate": (i, P),
            "vref_model_free": (None, P),
            "vref_scene_config": (P, i, C.POINTER(P), u32, u64, i, i),
            "vref_scene_evaluate": (i, P, d),
            "vref_scene_mark_clean": (i, P),
            "vref_scene_set_camera_dirty": (i, P, i),
            "vref_scene_set_camera": (i, P, P, P, P, d, i, i),
            "vref_scene_get_object": (i, P, i, C.POINTER(C.c_int32), C.POINTER(d), C.POINTER(i)),
            "vref_scene_set_object": (i, P, i, C.POINTER(d), i),
            "vref_scene_free": (None, P),
            "vref_hbo_create": (P, i, i),
            "vref_hbo_free": (None, P),
            "vref_hbo_records": (i, P, P),
            "vref_hbo_set_record": (i, P, i, i, P),
            "vref_render": (i, P, i, i, i, P, P, C.POINTER(u64), C.POINTER(d)),
            "vref_dump": (i, P, i, i, i, i, i, P, P),
            "vref_render_rows": (i, P, i, i, i, P, C.POINTER(d)),
            "vref_explain": (i, P, i, i, P, P, C.c_char_p, C.c_size_t),
            "vref_classify": (i, P, i, i, P, P, d, P),
            "vref_classify_rules": (i, P, i, i, P, P, d, P),
            "vref_traverse": (i, P, P, u32, P, i),
            "vref_dda_random": (i, u64, u32, d, P, u32, P, P, P),
            "vref_primary_ray": (i, P, i, i, C.POINTER(d)),
            "vref_hardware_threads": (i,),
        }
        for name, (res, *args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _err():
    return lib().vref_last_error().decode()


def _ok(rc, what):
    if rc != 0:
        raise RuntimeError(f"oracle {what}: {_err()}")


class RefModel:
    def __init__(self, h):
        if not h:
            raise RuntimeError(_err())
        self._h = C.c_void_p(h)

    @classmethod
    def from_bytes(cls, data: bytes):
        buf = C.create_string_buffer(data, len(data))
        return cls(lib().vref_model_deserialize(buf, len(data)))

    @classmethod
    def load(cls, path: str):
        """The reference load_svo (svo.cpp) of a .svo file."""
        return cls(lib().vref_model_load(path.encode()))

    @classmethod
    def dense_sphere(cls, depth):
        return cls(lib().vref_model_dense_sphere(depth))

    @classmethod
    def shell_grid(cls, depth):
        return cls(lib().vref_model_shell_grid(depth))

    @classmethod
    def random(cls, seed, depth, fill):
        return cls(lib().vref_model_random(seed, depth, fill))

    @classmethod
    def from_grid(cls, words, depth, color_mode=0, color_rgba=0xFFC8C8C8):
        """The reference build_from_grid of a VoxelGrid bitset (numpy uint64 words)."""
        import numpy as np
        w = np.ascontiguousarray(words, dtype=np.uint64)
        return cls(lib().vref_model_from_grid(w.ctypes.data, depth, color_mode, color_rgba))

    def violations(self) -> int:
        return lib().vref_model_validate(self._h)

    def serialize(self) -> bytes:
        n = lib().vref_model_serialize(self._h, None, 0)
        buf = C.create_string_buffer(n)
        lib().vref_model_serialize(self._h, buf, n)
        return buf.raw

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.vref_model_free(self._h)
            self._h = None


class RefHitBuffer:
    def __init__(self, w, h):
        self._h = C.c_void_p(lib().vref_hbo_create(w, h))
        self.width, self.height = w, h

    def records(self):
        """The reference HitBuffer's records (HBO_DTYPE, height x width)."""
        import numpy as np
        from paper_1911_06001_b200._abi import HBO_DTYPE
        out = np.zeros((self.height, self.width), HBO_DTYPE)
        lib().vref_hbo_records(self._h, out.ctypes.data)
        return out

    def set_record(self, x, y, rec):
        import numpy as np
        from paper_1911_06001_b200._abi import HBO_DTYPE
        r = np.array(rec, HBO_DTYPE)
        lib().vref_hbo_set_record(self._h, x, y, r.ctypes.data)

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.vref_hbo_free(self._h)


class RefScene:
    def __init__(self, cfg, models, seed=0, width=0, height=0):
        self.models = list(models)
        arr = (C.c_void_p * len(self.models))(*[m._h for m in self.models])
        h = lib().vref_scene_config(cfg, arr, len(self.models), seed, width, height)
        if not h:
            raise RuntimeError(_err())
        self._h = C.c_void_p(h)
        dw, dh = CONFIG_SIZES[cfg]
        self.width, self.height = width or dw, height or dh

    def evaluate(self, t):
        _ok(lib().vref_scene_evaluate(self._h, t), "evaluate_animation")

    def mark_clean(self):
        lib().vref_scene_mark_clean(self._h)

    def set_camera_dirty(self, dirty):
        lib().vref_scene_set_camera_dirty(self._h, 1 if dirty else 0)

    def get_object(self, i):
        oid, tf, dirty = C.c_int32(), (C.c_double * 15)(), C.c_int()
        _ok(lib().vref_scene_get_object(self._h, i, C.byref(oid), tf, C.byref(dirty)), "get_object")
        return oid.value, list(tf), bool(dirty.value)

    def set_camera(self, position, look_at, up=(0.0, 1.0, 0.0), fov_deg=60.0, width=None, height=None):
        w, h = width or self.width, height or self.height
        P3 = C.c_double * 3
        _ok(lib().vref_scene_set_camera(self._h, P3(*position), P3(*look_at), P3(*up), float(fov_deg), w, h),
            "set_camera")
        self.width, self.height = w, h

    def set_object(self, i, transform15, dirty):
        tf = (C.c_double * 15)(*transform15)
        _ok(lib().vref_scene_set_object(self._h, i, tf, 1 if dirty else 0), "set_object")

    def render(self, culling=True, sorting=True, threads=0, hbo=None):
        """Reference render_frame: (rgb HxWx3, FrameStats dict incl. render_ms)."""
        W, H = self.width, self.height
        img = np.zeros((H, W, 3), np.uint8)
        fs = (C.c_uint64 * 4)()
        ms = C.c_double()
        _ok(lib().vref_render(self._h, int(culling), int(sorting), threads, hbo._h if hbo else None,
                              img.ctypes.data, fs, C.byref(ms)), "render_frame")
        return img, {"rays": fs[0], "sphere_tests": fs[1], "svo_traversals": fs[2], "pixels_reused": fs[3],
                     "render_ms": ms.value}

    def render_rows(self, a, b, threads=0, rgb=True):
        """Reference per-pixel pipeline (culling+sorting) over rows [a, b): (rgb, wall ms)."""
        img = np.zeros((b - a, self.width, 3), np.uint8) if rgb else None
        ms = C.c_double()
        _ok(lib().vref_render_rows(self._h, threads, a, b, img.ctypes.data if rgb else None, C.byref(ms)),
            "render_rows")
        return img, ms.value

    def dump(self, culling=True, sorting=True, threads=0, rows=None):
        """Per-pixel oracle AOVs (+ RGB) for rows [a, b)."""
        W, H = self.width, self.height
        a, b = rows if rows else (0, H)
        aov = np.zeros((b - a, W), AOV_DTYPE)
        rgb = np.zeros((b - a, W, 3), np.uint8)
        _ok(lib().vref_dump(self._h, int(culling), int(sorting), threads, a, b, aov.ctypes.data, rgb.ctypes.data),
            "dump")
        return aov, rgb

    def classify(self, oracle_aov, gpu_aov, t_rel=1e-6, rows=None):
        a, b = rows if rows else (0, self.height)
        o = np.ascontiguousarray(oracle_aov, AOV_DTYPE)
        g = np.ascontiguousarray(gpu_aov, AOV_DTYPE)
        cls = np.zeros((b - a, self.width), np.uint8)
        _ok(lib().vref_classify(self._h, a, b, o.ctypes.data, g.ctypes.data, t_rel, cls.ctypes.data), "classify")
        return cls

    def classify_rules(self, oracle_aov, gpu_aov, t_rel=1e-6, rows=None):
        """Per-pixel rule code (RULES) of each FP32-vs-oracle difference."""
        a, b = rows if rows else (0, self.height)
        o = np.ascontiguousarray(oracle_aov, AOV_DTYPE)
        g = np.ascontiguousarray(gpu_aov, AOV_DTYPE)
        out = np.zeros((b - a, self.width), np.uint8)
        _ok(lib().vref_classify_rules(self._h, a, b, o.ctypes.data, g.ctypes.data, t_rel, out.ctypes.data),
            "classify_rules")
        return out

    def explain(self, px, py, oracle_rec, gpu_rec):
        o = np.ascontiguousarray(np.array([oracle_rec], AOV_DTYPE))
        g = np.ascontiguousarray(np.array([gpu_rec], AOV_DTYPE))
        buf = C.create_string_buffer(8192)
        _ok(lib().vref_explain(self._h, px, py, o.ctypes.data, g.ctypes.data, buf, 8192), "explain")
        return buf.value.decode()

    def primary_ray(self, px, py):
        o6 = (C.c_double * 6)()
        _ok(lib().vref_primary_ray(self._h, px, py, o6), "primary_ray")
        return list(o6)

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.vref_scene_free(self._h)


def rule_histogram(rules, hit_mask=None) -> dict:
    """{rule name: pixel count} of the non-matching pixels (+ the hit-pixel total)."""
    vals, counts = np.unique(rules, return_counts=True)
    h = {RULES.get(int(v), str(int(v))): int(c) for v, c in zip(vals, counts) if v != 0}
    if hit_mask is not None:
        h["hit_pixels"] = int(hit_mask.sum())
    return h


def traverse(model: RefModel, rays, with_fetches=False):
    rays = np.ascontiguousarray(rays, RAY_DTYPE)
    out = np.zeros(len(rays), TRAV_DTYPE)
    _ok(lib().vref_traverse(model._h, rays.ctypes.data, len(rays), out.ctypes.data, int(with_fetches)), "traverse")
    return out


def dda_random(seed, depth, fill, rays):
    rays = np.ascontiguousarray(rays, RAY_DTYPE)
    n = len(rays)
    hit = np.zeros(n, np.int32)
    vox = np.zeros((n, 3), np.uint32)
    t = np.zeros(n, np.float64)
    _ok(lib().vref_dda_random(seed, depth, fill, rays.ctypes.data, n, hit.ctypes.data, vox.ctypes.data,
                              t.ctypes.data), "dda")
    return hit, vox, t


def hardware_threads() -> int:
    return lib().vref_hardware_threads()
