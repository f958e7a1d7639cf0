"""TEST INFRASTRUCTURE — ctypes binding of the plain-C restatement (oracle/voxanim_oracle.c).

Only tests/ use it. Models are passed as their .svo bytes (parsed here with
numpy), objects as the 15 doubles of RigidTransform, the camera as the values
of voxanim::Camera.
"""
from __future__ import annotations

import ctypes as C
import os
import struct

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libvoxanim_oracle.so")

AOV_DTYPE = np.dtype(
    [("t", "<f8"), ("object_id", "<i4"), ("node_index", "<u4"), ("attr_index", "<u4"), ("voxel", "<u4", (3,)),
     ("level", "u1"), ("kind", "u1"), ("entry_axis", "u1"), ("pad0", "u1"), ("traversals", "<u4"),
     ("node_fetches", "<u4"), ("pad1", "<u4")]
)
NODE_DTYPE = np.dtype([("child_base", "<u4"), ("attr_base", "<u4"), ("valid", "u1"), ("leaf", "u1"),
                       ("pad", "u1", (2,))])


class _Model(C.Structure):
    _fields_ = [("nodes", C.c_void_p), ("attrs", C.c_void_p), ("depth", C.c_uint32)]


class _Object(C.Structure):
    _fields_ = [("id", C.c_int32), ("model", C.c_int32), ("R", C.c_double * 9), ("t", C.c_double * 3),
                ("s", C.c_double * 3)]


class _Camera(C.Structure):
    _fields_ = [("pos", C.c_double * 3), ("C", C.c_double * 9), ("fov_deg", C.c_double), ("width", C.c_int32),
                ("height", C.c_int32), ("background", C.c_uint8 * 3)]


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            import subprocess

            subprocess.run(["make", "-C", HERE, "_build/libvoxanim_oracle.so"], check=True,
                           capture_output=True)
        L = C.CDLL(LIB_PATH)
        L.vo_render.restype = None
        L.vo_render.argtypes = [C.POINTER(_Camera), C.POINTER(_Object), C.c_int, C.POINTER(_Model), C.c_int, C.c_int,
                                C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        _LIB = L
    return _LIB


def parse_svo(data: bytes):
    """(depth, nodes[NODE_DTYPE], attrs[uint8 x4]) of an SVOA v1 stream (svo.cpp:205-229)."""
    magic, version, depth, nn, na = struct.unpack_from("<4sIIII", data, 0)
    assert magic == b"SVOA" and version == 1
    nodes = np.frombuffer(data, NODE_DTYPE, nn, 20)
    attrs = np.frombuffer(data, np.uint8, 4 * na, 20 + 12 * nn)
    return depth, np.ascontiguousarray(nodes), np.ascontiguousarray(attrs)


def render(frame_desc, objects, model_bytes, object_model, culling=True, sorting=True, rows=None):
    """objects: [(id, tf15)], object_model: model index per object (-1: none).
    Returns (rgb HxWx3, aov HxW) for rows [a, b)."""
    keep = [parse_svo(b) for b in model_bytes]
    models = (_Model * max(1, len(keep)))()
    for i, (depth, nodes, attrs) in enumerate(keep):
        models[i].nodes = nodes.ctypes.data
        models[i].attrs = attrs.ctypes.data
        models[i].depth = depth
    objs = (_Object * max(1, len(objects)))()
    for i, (oid, tf) in enumerate(objects):
        objs[i].id = oid
        objs[i].model = object_model[i]
        objs[i].R[:] = tf[0:9]
        objs[i].t[:] = tf[9:12]
        objs[i].s[:] = tf[12:15]
    cam = _Camera()
    c = frame_desc.camera
    cam.pos[:] = list(c.position)
    cam.C[:] = list(c.orientation)
    cam.fov_deg = c.vertical_fov_deg
    cam.width, cam.height = c.width, c.height
    cam.background[:] = list(frame_desc.background)
    a, b = rows if rows else (0, c.height)
    rgb = np.zeros((b - a, c.width, 3), np.uint8)
    aov = np.zeros((b - a, c.width), AOV_DTYPE)
    lib().vo_render(C.byref(cam), objs, len(objects), models, int(culling), int(sorting), a, b, rgb.ctypes.data,
                    aov.ctypes.data)
    return rgb, aov
