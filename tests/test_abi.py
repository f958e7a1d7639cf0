"""CPU: the drop-in boundary itself.

* libvxa.so exports every symbol include/vxa.h declares (and libvoxanim.so every
  symbol of include/voxanim_capi.h), parsed from the headers, not hard-coded;
* the ctypes mirrors have the C layouts;
* without a GPU the product fails loudly (DeviceError / VXA_ERR_NO_DEVICE) —
  it never renders through a CPU fallback;
* the library's voxanim:: symbols and the reference oracle's never interpose
  (the oracle exports only its vref_* C functions).
"""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_1911_06001_b200 as vx
from paper_1911_06001_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions(name):
    text = open(os.path.join(ROOT, "include", name)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vx[an]_[a-z0-9_]+)\s*\(", text)))


def exported(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_vxa_exports_every_declared_symbol():
    declared = header_functions("vxa.h")
    assert len(declared) >= 20
    syms = exported(os.path.join(_abi.LIB_DIR, "libvxa.so"))
    missing = [f for f in declared if f not in syms]
    assert not missing, missing
    assert sorted(_abi.VXA_SYMBOLS) == declared


def test_capi_exports_every_declared_symbol():
    declared = header_functions("voxanim_capi.h")
    syms = exported(os.path.join(_abi.LIB_DIR, "libvoxanim.so"))
    missing = [f for f in declared if f not in syms]
    assert not missing, missing
    assert sorted(_abi.VXN_SYMBOLS) == declared


def test_libvoxanim_exports_the_reference_cpp_api():
    syms = exported(os.path.join(_abi.LIB_DIR, "libvoxanim.so"))
    demangled = subprocess.run(["c++filt"], input="\n".join(syms), capture_output=True, text=True).stdout
    for fn in ["voxanim::render_frame(voxanim::Scene const&, voxanim::RenderOptions const&, voxanim::FrameStats&)",
               "voxanim::traverse(voxanim::SvoModel const&, voxanim::Ray const&, voxanim::OctreeBounds const&)",
               "voxanim::load_svo(std::filesystem::__cxx11::path const&)",
               "voxanim::build_from_grid(voxanim::VoxelGrid const&, unsigned int)",
               "voxanim::evaluate_animation(voxanim::Scene&, double)"]:
        assert fn in demangled, fn


def test_oracle_exports_only_c_entry_points():
    from oracle import ref

    syms = exported(ref.LIB_PATH)
    assert not [s for s in syms if "voxanim" in s]
    assert "vref_render" in syms and "vref_dump" in syms


def test_struct_layouts():
    assert C.sizeof(_abi.vxa_instance) == 136
    assert C.sizeof(_abi.vxa_hit_record) == 48
    assert C.sizeof(_abi.vxa_pixel_aov) == 48
    assert C.sizeof(_abi.vxa_traverse_hit) == 96
    assert C.sizeof(_abi.vxa_stats) == 88
    assert vx.vxa().vxa_abi_version() == 1


def test_tile_owner_partition_is_complete_and_round_robin():
    lib = vx.vxa()
    W, H = 3840, 2160
    for world in (1, 2, 4, 8):
        counts = [0] * world
        for y in range(0, H, 16):
            for x in range(0, W, 16):
                r = lib.vxa_tile_owner(x, y, W, H, world)
                assert 0 <= r < world
                counts[r] += 1
        assert min(counts) > 0
        assert max(counts) - min(counts) <= 0.05 * max(counts) + 64  # round-robin balance
    assert lib.vxa_tile_owner(W, 0, W, H, 2) == -1


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device failure path")
def test_no_device_fails_loudly():
    lib = vx.vxa()
    ctx = C.c_void_p()
    rc = lib.vxa_create(0, C.byref(ctx))
    assert rc == _abi.VXA_ERR_NO_DEVICE
    assert lib.vxa_last_error()
    model = vx.Model.procedural(3)
    scene = vx.Scene(vx.config.C1, [model], 0, 8, 8)
    with pytest.raises(vx.VoxanimError, match="no CUDA device"):
        scene.render()
    with pytest.raises(vx.VoxanimError, match="no CUDA device"):
        vx.traverse(model, __import__("numpy").zeros(1, vx.RAY_DTYPE))
