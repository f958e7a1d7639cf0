// voxanim-b200: sparse procedural SVO content (new API, not in the reference).
//
// The reference can only build models from a dense VoxelGrid, capped at
// depth 10 (proj/src/ingest.cpp:15,271-274) and costing ~48 s / 15 GB at
// depth 10. The benchmark configurations need depth 10 and 11, so this
// builder evaluates the reference's sphere occupancy rule
// (ingest.cpp:195-211) analytically per cube and emits the identical
// breadth-first layout and PositionHash colours (ingest.cpp:24-29,74-84);
// for depth <= 10 its serialize() output is byte-identical to
// build_from_grid(gen_primitive(Sphere, depth), depth) (tests/test_procedural.py).
#pragma once

#include <cstdint>

#include "voxanim/svo.hpp"

namespace voxanim {

enum class ProceduralShape : std::uint8_t {
    SolidSphere, // voxel set iff (x+.5-c)^2+(y+.5-c)^2+(z+.5-c)^2 <= c^2, c = 2^depth/2
    ShellSphere, // solid voxels on the grid boundary or with a 6-neighbour outside the solid
};

SvoModel build_procedural(ProceduralShape shape, std::uint32_t depth, ColorSpec colors = {});

// Dense reference grid of the same shape (depth <= 10), for layout checks.
VoxelGrid procedural_grid(ProceduralShape shape, std::uint32_t depth, ColorSpec colors = {});

} // namespace voxanim
