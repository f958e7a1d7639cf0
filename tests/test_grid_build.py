"""CPU: build_from_grid on caller-supplied VoxelGrid bitsets — the product's
host builder (level-synchronous BFS, csrc/host/svo.cpp) against the reference's
own build_from_grid (proj/src/svo.cpp:52-132, compiled in oracle/_ref) on the
same grid: serialized streams identical byte for byte, for every colour mode
(ingest.cpp:24-29,67-85), the reference primitives (ingest.cpp:193-266) and the
edge cases (empty grid, full grid, one voxel, depth 1). These grids are also
the inputs of the device-builder parity tests (test_gpu_builder.py)."""
import numpy as np
import pytest

import paper_1911_06001_b200 as vx
from oracle import ref

MODES = [(0, 0xFFC8C8C8), (1, 0xFFC8C8C8), (2, 0x80402010)]


def random_grid(seed, depth, fill):
    n = 1 << depth
    rng = np.random.default_rng(seed)
    bits = rng.random(n ** 3) < fill
    return pack(bits)


def pack(bits):
    """x-major boolean array (index (x*n + y)*n + z) -> VoxelGrid words."""
    bits = np.asarray(bits, bool).ravel()
    pad = (-bits.size) % 64
    b = np.concatenate([bits, np.zeros(pad, bool)]).reshape(-1, 64)
    return (b.astype(np.uint64) << np.arange(64, dtype=np.uint64)).sum(axis=1, dtype=np.uint64)


def edge_grids():
    yield "empty d3", np.zeros(8, np.uint64), 3
    yield "full d3", np.full(8, np.uint64(0xFFFFFFFFFFFFFFFF)), 3
    one = np.zeros(8 ** 3, bool)
    one[(5 * 8 + 2) * 8 + 7] = True
    yield "one voxel d3", pack(one), 3
    yield "full d1", np.array([0xFF], np.uint64), 1
    yield "one voxel d1", np.array([0x20], np.uint64), 1
    yield "empty d1", np.array([0], np.uint64), 1


def same_model(words, depth, mode=0, rgba=0xFFC8C8C8, device=False):
    ours = vx.Model.from_grid(words, depth, mode, rgba, device=device).serialize()
    theirs = ref.RefModel.from_grid(words, depth, mode, rgba).serialize()
    return ours == theirs, len(ours)


@pytest.mark.parametrize("mode,rgba", MODES)
def test_random_grids_match_reference(mode, rgba):
    for seed, depth, fill in [(1, 2, 0.5), (2, 4, 0.1), (3, 5, 0.02), (4, 6, 0.3), (5, 3, 0.9)]:
        ok, n = same_model(random_grid(seed, depth, fill), depth, mode, rgba)
        assert ok, (seed, depth, fill, mode)


def test_edge_grids_match_reference():
    for name, words, depth in edge_grids():
        ok, _ = same_model(words, depth)
        assert ok, name


@pytest.mark.parametrize("kind", sorted(vx.PRIMITIVES))
def test_primitives_match_reference(kind):
    for depth in (1, 3, 5):
        words, grid_depth = vx.grid_primitive(kind, depth)
        ok, _ = same_model(words, grid_depth, 1)
        assert ok, (kind, depth)


def test_from_grid_argument_errors():
    with pytest.raises(vx.VoxanimError):
        vx.Model.from_grid(np.zeros(3, np.uint64), 3, device=False)  # wrong word count
    with pytest.raises(vx.VoxanimError):
        vx.Model.from_grid(np.zeros(1, np.uint64), 1, color_mode=7, device=False)
