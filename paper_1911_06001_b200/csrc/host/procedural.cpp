// Sparse procedural sphere SVOs (solid and one-voxel shell) at any depth <= 16.
//
// Occupancy is evaluated per cube in doubled integer coordinates: with
// c = n/2, voxel v is solid iff sum_a (2 v_a + 1 - n)^2 <= n^2, which is the
// reference's FP64 test (proj/src/ingest.cpp:195-211) exactly, because the
// reference's half-integer differences and their squares are exact doubles.
// A cube holds a solid voxel iff the per-axis minimum |u| gives sum <= n^2;
// every voxel of a box is solid iff the per-axis maximum |u| does (the
// squared distance is separable and convex). A cube holds a shell voxel iff
// it holds a solid voxel and is not "interior": interior means the cube,
// grown by one voxel along each axis separately, stays inside the grid and
// all-solid (a path argument shows any non-interior cube with a solid voxel
// contains a solid voxel with a non-solid or out-of-grid 6-neighbour).
#include "voxanim/procedural.hpp"

#include <algorithm>
#include <cstdlib>

#include "bfs_builder.hpp"

namespace voxanim {

namespace {

using i64 = std::int64_t;

struct SphereLattice {
    i64 n; // 2^depth

    // min / max of |2v + 1 - n| over v in [a, b]
    i64 min_abs(i64 a, i64 b) const {
        const i64 lo = 2 * a + 1 - n, hi = 2 * b + 1 - n;
        if (lo > 0) return lo;
        if (hi < 0) return -hi;
        return 1; // odd values straddling zero
    }
    i64 max_abs(i64 a, i64 b) const { return std::max(std::llabs(2 * a + 1 - n), std::llabs(2 * b + 1 - n)); }

    bool any_solid(const i64 lo[3], const i64 hi[3]) const {
        i64 s = 0;
        for (int k = 0; k < 3; ++k) {
            const i64 m = min_abs(lo[k], hi[k]);
            s += m * m;
        }
        return s <= n * n;
    }
    bool all_solid(const i64 lo[3], const i64 hi[3]) const {
        i64 s = 0;
        for (int k = 0; k < 3; ++k) {
            const i64 m = max_abs(lo[k], hi[k]);
            s += m * m;
        }
        return s <= n * n;
    }
    bool interior(const i64 lo[3], const i64 hi[3]) const {
        for (int a = 0; a < 3; ++a) {
            i64 glo[3] = {lo[0], lo[1], lo[2]}, ghi[3] = {hi[0], hi[1], hi[2]};
            --glo[a];
            ++ghi[a];
            if (glo[a] < 0 || ghi[a] > n - 1) return false;
            if (!all_solid(glo, ghi)) return false;
        }
        return true;
    }
    bool occupied(ProceduralShape shape, std::uint32_t depth, std::uint32_t level, std::uint32_t x, std::uint32_t y,
                  std::uint32_t z) const {
        const i64 side = i64{1} << (depth - level);
        const i64 lo[3] = {x * side, y * side, z * side};
        const i64 hi[3] = {lo[0] + side - 1, lo[1] + side - 1, lo[2] + side - 1};
        if (!any_solid(lo, hi)) return false;
        return shape == ProceduralShape::SolidSphere || !interior(lo, hi);
    }
};

void check_depth(std::uint32_t depth, std::uint32_t cap) {
    if (depth < 1 || depth > cap)
        throw ValidationError("procedural depth must be in [1, " + std::to_string(cap) + "], got " +
                              std::to_string(depth));
}

} // namespace

SvoModel build_procedural(ProceduralShape shape, std::uint32_t depth, ColorSpec colors) {
    check_depth(depth, 16);
    const SphereLattice s{i64{1} << depth};
    const std::uint32_t res = 1u << depth;
    return detail::build_breadth_first(
        depth,
        [&](std::uint32_t L, std::uint32_t x, std::uint32_t y, std::uint32_t z) {
            return s.occupied(shape, depth, L, x, y, z);
        },
        [&](std::uint32_t x, std::uint32_t y, std::uint32_t z) { return voxel_color(colors, res, x, y, z); });
}

VoxelGrid procedural_grid(ProceduralShape shape, std::uint32_t depth, ColorSpec colors) {
    check_depth(depth, 10);
    const SphereLattice s{i64{1} << depth};
    const std::uint32_t n = 1u << depth;
    VoxelGrid g(n, colors);
    for (std::uint32_t x = 0; x < n; ++x)
        for (std::uint32_t y = 0; y < n; ++y)
            for (std::uint32_t z = 0; z < n; ++z)
                if (s.occupied(shape, depth, depth, x, y, z)) g.set(x, y, z);
    return g;
}

} // namespace voxanim
