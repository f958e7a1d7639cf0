"""ctypes mirror of include/vxa.h and include/voxanim_capi.h.

Python is plumbing here: tests and bench.py drive the native libraries
(lib/libvxa.so — CUDA layer + C ABI; lib/libvoxanim.so — the drop-in
voxanim:: C++ API) through these declarations. There is no Python compute
path and no fallback: if a library is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

# VOXANIM_LIB_DIR selects an alternative build (tuning experiments); default: the in-tree lib/.
LIB_DIR = os.environ.get("VOXANIM_LIB_DIR") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")

VXA_OK, VXA_ERR_INVALID, VXA_ERR_MODEL, VXA_ERR_CUDA, VXA_ERR_OOM, VXA_ERR_NO_DEVICE = range(6)
VXA_FP32, VXA_FP64 = 0, 1
VXA_SYNC_DEVICE, VXA_SYNC_HOST = 0, 1


class vxa_camera(C.Structure):
    _fields_ = [
        ("position", C.c_double * 3),
        ("orientation", C.c_double * 9),
        ("vertical_fov_deg", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
    ]


class vxa_instance(C.Structure):
    _fields_ = [
        ("model", C.c_uint32),
        ("id", C.c_int32),
        ("rotation", C.c_double * 9),
        ("translation", C.c_double * 3),
        ("scale", C.c_double * 3),
        ("dirty", C.c_uint8),
        ("pad", C.c_uint8 * 7),
    ]


class vxa_hit_record(C.Structure):
    _fields_ = [
        ("color", C.c_uint8 * 4),
        ("pad0", C.c_uint8 * 4),
        ("normal", C.c_double * 3),
        ("t", C.c_double),
        ("object_id", C.c_int32),
        ("kind", C.c_uint8),
        ("pad1", C.c_uint8 * 3),
    ]


class vxa_frame_desc(C.Structure):
    _fields_ = [
        ("camera", vxa_camera),
        ("background", C.c_uint8 * 3),
        ("culling", C.c_uint8),
        ("sorting", C.c_uint8),
        ("precision", C.c_uint8),
        ("camera_dirty", C.c_uint8),
        ("pad0", C.c_uint8),
        ("tile_rank", C.c_int32),
        ("tile_world", C.c_int32),
        ("hbo", C.POINTER(vxa_hit_record)),
        ("hbo_device", C.c_uint32),
        ("pad1", C.c_uint32),
    ]


class vxa_stats(C.Structure):
    _fields_ = [
        ("rays", C.c_uint64),
        ("sphere_tests", C.c_uint64),
        ("svo_traversals", C.c_uint64),
        ("pixels_reused", C.c_uint64),
        ("node_fetches", C.c_uint64),
        ("leaf_hits", C.c_uint64),
        ("kernel_launches", C.c_uint64),
        ("gpu_ms", C.c_double),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("frames", C.c_uint64),
    ]


class vxa_pixel_aov(C.Structure):
    _fields_ = [
        ("t", C.c_double),
        ("object_id", C.c_int32),
        ("node_index", C.c_uint32),
        ("attr_index", C.c_uint32),
        ("voxel", C.c_uint32 * 3),
        ("level", C.c_uint8),
        ("kind", C.c_uint8),
        ("entry_axis", C.c_uint8),
        ("pad0", C.c_uint8),
        ("traversals", C.c_uint32),
        ("node_fetches", C.c_uint32),
        ("pad1", C.c_uint32),
    ]


class vxa_local_ray(C.Structure):
    _fields_ = [
        ("origin", C.c_double * 3),
        ("direction", C.c_double * 3),
        ("half_extent", C.c_double * 3),
    ]


class vxa_traverse_hit(C.Structure):
    _fields_ = [
        ("t_hit", C.c_double),
        ("t_enter", C.c_double),
        ("t_exit", C.c_double),
        ("normal_local", C.c_double * 3),
        ("attribute", C.c_uint8 * 4),
        ("attr_index", C.c_uint32),
        ("node_index", C.c_uint32),
        ("leaf_path", C.c_uint8 * 16),
        ("path_len", C.c_uint8),
        ("hit", C.c_uint8),
        ("pad", C.c_uint16),
        ("node_fetches", C.c_uint32),
        ("log_count", C.c_uint32),
        ("log_total", C.c_uint32),
    ]


class vxa_visit(C.Structure):
    _fields_ = [("t_enter", C.c_double), ("level", C.c_uint8), ("leaf", C.c_uint8), ("pad", C.c_uint8 * 6)]


assert C.sizeof(vxa_instance) == 136
assert C.sizeof(vxa_hit_record) == 48
assert C.sizeof(vxa_pixel_aov) == 48
assert C.sizeof(vxa_local_ray) == 72
assert C.sizeof(vxa_traverse_hit) == 96

# numpy dtypes with the same layouts (for bulk AOV / ray arrays)
try:
    import numpy as np

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
    # voxanim::HitRecord / vxa_hit_record (48 bytes)
    HBO_DTYPE = np.dtype(
        [("color", "u1", (4,)), ("pad0", "u1", (4,)), ("normal", "<f8", (3,)), ("t", "<f8"), ("object_id", "<i4"),
         ("kind", "u1"), ("pad1", "u1", (3,))]
    )
    assert AOV_DTYPE.itemsize == 48 and RAY_DTYPE.itemsize == 72 and TRAV_DTYPE.itemsize == 96
    assert HBO_DTYPE.itemsize == 48
except ImportError:  # pragma: no cover
    np = None

# Every symbol include/vxa.h declares (checked by tests/test_abi.py).
VXA_SYMBOLS = [
    "vxa_create", "vxa_destroy", "vxa_last_error", "vxa_abi_version", "vxa_device_info",
    "vxa_upload_model", "vxa_release_model", "vxa_model_info", "vxa_build_model", "vxa_model_download", "vxa_upload_svo",
    "vxa_model_counts",
    "vxa_hbo_create", "vxa_hbo_release", "vxa_hbo_download", "vxa_hbo_upload", "vxa_render", "vxa_submit", "vxa_submit_readback",
    "vxa_wait_readback", "vxa_synchronize", "vxa_stats_read", "vxa_stats_reset", "vxa_read_framebuffer",
    "vxa_host_register", "vxa_host_unregister", "vxa_timer_begin", "vxa_timer_end", "vxa_flush_l2", "vxa_stream_delay", "vxa_stream",
    "vxa_fb_export", "vxa_fb_import", "vxa_tile_owner", "vxa_tiles_count", "vxa_tiles_pack", "vxa_tiles_unpack", "vxa_traverse",
    "vxa_sync_export", "vxa_sync_import", "vxa_sync_configure", "vxa_frame_open", "vxa_frame_close", "vxa_sync_status",
    "vxa_framebuffer_readback",
]
VXN_SYMBOLS = [
    "vxn_last_error", "vxn_model_procedural", "vxn_model_dense_sphere", "vxn_model_random", "vxn_model_full_cube",
    "vxn_model_from_grid", "vxn_grid_primitive", "vxn_model_deserialize", "vxn_model_save", "vxn_scene_load", "vxn_model_serialize", "vxn_model_info", "vxn_model_validate", "vxn_model_free",
    "vxn_scene_config", "vxn_scene_evaluate", "vxn_scene_mark_clean", "vxn_scene_set_camera_dirty",
    "vxn_scene_set_camera",
    "vxn_scene_object_count", "vxn_scene_get_object", "vxn_scene_set_object", "vxn_scene_export", "vxn_scene_free", "vxn_scene_submit", "vxn_scene_stream",
    "vxn_hbo_create", "vxn_hbo_free", "vxn_hbo_records", "vxn_hbo_set_record", "vxn_render", "vxn_scene_render_image",
    "vxn_traverse", "vxn_context",
]

P = C.c_void_p


def _declare(lib, name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)


def load_vxa(path: str | None = None) -> C.CDLL:
    path = path or os.path.join(LIB_DIR, "libvxa.so")
    if not os.path.exists(path):
        raise RuntimeError(f"voxanim-b200: CUDA library {path} is missing; run __graft_entry__.build()")
    lib = C.CDLL(path, mode=C.RTLD_LOCAL)
    i, u32, u64, d = C.c_int, C.c_uint32, C.c_uint64, C.c_double
    _declare(lib, "vxa_create", i, i, C.POINTER(P))
    _declare(lib, "vxa_destroy", i, P)
    _declare(lib, "vxa_last_error", C.c_char_p)
    _declare(lib, "vxa_abi_version", i)
    _declare(lib, "vxa_device_info", i, P, C.POINTER(i), C.POINTER(i), C.c_char_p, C.c_size_t)
    _declare(lib, "vxa_upload_model", i, P, P, u32, P, u32, u32, C.POINTER(u32))
    _declare(lib, "vxa_release_model", i, P, u32)
    _declare(lib, "vxa_model_info", i, P, u32, C.POINTER(u64), C.POINTER(u32))
    _declare(lib, "vxa_build_model", i, P, P, u32, u32, u32, C.POINTER(u32), C.POINTER(u64), C.POINTER(u64))
    _declare(lib, "vxa_model_download", i, P, u32, P, u64, P, u64)
    _declare(lib, "vxa_upload_svo", i, P, P, C.c_size_t, C.POINTER(u32), C.POINTER(C.c_int32))
    _declare(lib, "vxa_model_counts", i, P, u32, C.POINTER(u32), C.POINTER(u64), C.POINTER(u64))
    _declare(lib, "vxa_render", i, P, C.POINTER(vxa_frame_desc), C.POINTER(vxa_instance), u32, P, P,
             C.POINTER(vxa_stats))
    _declare(lib, "vxa_submit", i, P, C.POINTER(vxa_frame_desc), C.POINTER(vxa_instance), u32)
    _declare(lib, "vxa_submit_readback", i, P, C.POINTER(vxa_frame_desc), C.POINTER(vxa_instance), u32, P,
             C.POINTER(u64))
    _declare(lib, "vxa_wait_readback", i, P, u64)
    _declare(lib, "vxa_hbo_create", i, P, C.c_int32, C.c_int32, C.POINTER(u32))
    _declare(lib, "vxa_hbo_release", i, P, u32)
    _declare(lib, "vxa_hbo_download", i, P, u32, P)
    _declare(lib, "vxa_hbo_upload", i, P, u32, P)
    _declare(lib, "vxa_synchronize", i, P)
    _declare(lib, "vxa_stats_read", i, P, C.POINTER(vxa_stats))
    _declare(lib, "vxa_stats_reset", i, P)
    _declare(lib, "vxa_read_framebuffer", i, P, P, C.c_int32, C.c_int32)
    _declare(lib, "vxa_host_register", i, P, P, C.c_size_t)
    _declare(lib, "vxa_host_unregister", i, P, P)
    _declare(lib, "vxa_timer_begin", i, P)
    _declare(lib, "vxa_timer_end", i, P, C.POINTER(d))
    _declare(lib, "vxa_flush_l2", i, P)
    _declare(lib, "vxa_stream_delay", i, P, C.c_uint32)
    _declare(lib, "vxa_stream", P, P)
    _declare(lib, "vxa_fb_export", i, P, C.c_int32, C.c_int32, P)
    _declare(lib, "vxa_fb_import", i, P, C.c_int32, C.c_int32, P)
    _declare(lib, "vxa_traverse", i, P, u32, P, u32, u32, P, P, u32)
    _declare(lib, "vxa_tile_owner", C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32)
    _declare(lib, "vxa_tiles_count", i, i, i, i, i, C.POINTER(u32))
    _declare(lib, "vxa_tiles_pack", i, P, i, i, i, i, P)
    _declare(lib, "vxa_tiles_unpack", i, P, i, i, i, i, P)
    _declare(lib, "vxa_sync_export", i, P, C.c_int32, P)
    _declare(lib, "vxa_sync_import", i, P, C.c_int32, C.c_int32, P)
    _declare(lib, "vxa_sync_configure", i, P, C.c_int32, u32)
    _declare(lib, "vxa_frame_open", i, P)
    _declare(lib, "vxa_frame_close", i, P)
    _declare(lib, "vxa_sync_status", i, P, C.POINTER(C.c_int32))
    _declare(lib, "vxa_framebuffer_readback", i, P, C.c_int32, C.c_int32, P, C.POINTER(u64))
    return lib


def load_voxanim(path: str | None = None) -> C.CDLL:
    load_vxa()
    path = path or os.path.join(LIB_DIR, "libvoxanim.so")
    if not os.path.exists(path):
        raise RuntimeError(f"voxanim-b200: host library {path} is missing; run __graft_entry__.build()")
    lib = C.CDLL(path, mode=C.RTLD_LOCAL)
    i, u32, u64, d = C.c_int, C.c_uint32, C.c_uint64, C.c_double
    _declare(lib, "vxn_last_error", C.c_char_p)
    _declare(lib, "vxn_model_procedural", P, i, u32)
    _declare(lib, "vxn_model_dense_sphere", P, u32)
    _declare(lib, "vxn_model_random", P, u64, u32, d)
    _declare(lib, "vxn_model_full_cube", P)
    _declare(lib, "vxn_model_from_grid", P, P, u32, u32, u32, i)
    _declare(lib, "vxn_grid_primitive", C.c_int64, i, u32, P, C.c_size_t, C.POINTER(u32))
    _declare(lib, "vxn_model_deserialize", P, P, C.c_size_t)
    _declare(lib, "vxn_model_save", i, P, C.c_char_p)
    _declare(lib, "vxn_scene_load", P, C.c_char_p, i, i)
    _declare(lib, "vxn_model_serialize", C.c_int64, P, P, C.c_size_t)
    _declare(lib, "vxn_model_info", i, P, C.POINTER(u32), C.POINTER(u64), C.POINTER(u64))
    _declare(lib, "vxn_model_validate", i, P)
    _declare(lib, "vxn_model_free", None, P)
    _declare(lib, "vxn_scene_config", P, i, C.POINTER(P), u32, u64, i, i)
    _declare(lib, "vxn_scene_evaluate", i, P, d)
    _declare(lib, "vxn_scene_mark_clean", i, P)
    _declare(lib, "vxn_scene_set_camera_dirty", i, P, i)
    _declare(lib, "vxn_scene_set_camera", i, P, P, P, P, d, i, i)
    _declare(lib, "vxn_scene_object_count", i, P)
    _declare(lib, "vxn_scene_get_object", i, P, i, C.POINTER(C.c_int32), C.POINTER(d), C.POINTER(i))
    _declare(lib, "vxn_scene_set_object", i, P, i, C.POINTER(d), i)
    _declare(lib, "vxn_scene_export", i, P, C.POINTER(vxa_frame_desc), C.POINTER(vxa_instance), u32,
             C.POINTER(u32))
    _declare(lib, "vxn_scene_free", None, P)
    _declare(lib, "vxn_scene_submit", i, P, d, i, i, i, u32)
    _declare(lib, "vxn_scene_stream", i, P, d, i, P, C.POINTER(u64))
    _declare(lib, "vxn_scene_render_image", i, P, d, i, C.POINTER(d), P)
    _declare(lib, "vxn_hbo_create", P, i, i)
    _declare(lib, "vxn_hbo_free", None, P)
    _declare(lib, "vxn_hbo_records", i, P, P)
    _declare(lib, "vxn_hbo_set_record", i, P, i, i, P)
    _declare(lib, "vxn_render", i, P, i, i, i, P, P, P, C.POINTER(u64), C.POINTER(d), C.POINTER(vxa_stats))
    _declare(lib, "vxn_traverse", i, P, P, u32, P)
    _declare(lib, "vxn_context", P)
    return lib
