"""The reference's own doctest suites (proj/tests/test_*.cpp), compiled in place by
tests/cpp/Makefile with a doctest-compatible runner (tests/cpp/doctest.h):

* ref_*  -- against the reference sources: pins the oracle build (it must pass
  the reference's own 97 test cases, incl. the DDA equivalence, KATs, HBO
  transparency and thread determinism);
* our_*  -- the same sources against this repo's drop-in libvoxanim.so:
  test_math / test_svo / test_ingest / test_scene run on the CPU (model build,
  binvox, scene documents, animation); test_traversal / test_renderer drive
  traverse / trace_ray / render_frame through the CUDA kernels (GPU only).
"""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_bin")


def run_suite(name, env=None):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    res = subprocess.run([path], capture_output=True, text=True, timeout=1200, env=env)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    assert " 0 failed" in res.stdout
    return res.stdout


@pytest.mark.parametrize("suite", ["test_math", "test_svo", "test_ingest", "test_traversal", "test_scene",
                                   "test_renderer"])
def test_reference_suite_passes_against_the_oracle_build(suite):
    run_suite("ref_" + suite)


@pytest.mark.parametrize("suite", ["test_math", "test_svo", "test_ingest", "test_scene"])
def test_reference_suite_passes_against_our_library_cpu(suite):
    run_suite("our_" + suite)


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["test_traversal", "test_renderer"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_reference_suite_passes_against_our_library_gpu(gpu, suite, precision):
    env = dict(os.environ, VOXANIM_PRECISION=precision)
    run_suite("our_" + suite, env)
