// Level-synchronous breadth-first SVO construction.
//
// Produces exactly the node/attribute numbering of the reference builder
// (proj/src/svo.cpp:80-132): the reference pops nodes FIFO and, per popped
// node, walks octants 0..7 appending leaf attributes and enqueueing internal
// children; FIFO order means every level is finished before the next one
// starts, so emitting level L+1 as the concatenation (in level-L order) of
// each cube's non-empty children gives the same indices. child_base /
// attr_base are zeroed when a node has no internal / no leaf children.
//
// Unlike the reference (which recurses over all 8^depth sub-cubes of a dense
// grid) the cost here is proportional to the number of non-empty cubes, so
// sparse procedural content reaches depth 11+ (procedural.cpp).
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "voxanim/svo.hpp"

namespace voxanim::detail {

struct Cube {
    std::uint32_t x, y, z;
};

// occupied(level, x, y, z): does cube (x, y, z) of the 2^level lattice hold
// any voxel? colour(x, y, z): attribute of voxel (x, y, z) at full depth.
template <class Occupied, class Colour>
SvoModel build_breadth_first(std::uint32_t depth, Occupied&& occupied, Colour&& colour) {
    SvoModel model;
    model.depth = depth;
    model.nodes.emplace_back();
    std::vector<Cube> level_cubes{{0, 0, 0}};
    std::vector<Cube> next;
    std::uint32_t level_first = 0; // node index of level_cubes[0]
    for (std::uint32_t level = 0; level < depth; ++level) {
        const bool children_are_leaves = level + 1 == depth;
        next.clear();
        for (std::size_t i = 0; i < level_cubes.size(); ++i) {
            const Cube c = level_cubes[i];
            SvoNode node;
            const auto first_child = static_cast<std::uint32_t>(model.nodes.size());
            const auto first_attr = static_cast<std::uint32_t>(model.attributes.size());
            for (unsigned oct = 0; oct < 8; ++oct) {
                const Cube k{2 * c.x + ((oct >> 2) & 1u), 2 * c.y + ((oct >> 1) & 1u), 2 * c.z + (oct & 1u)};
                if (!occupied(level + 1, k.x, k.y, k.z)) continue;
                const auto bit = static_cast<std::uint8_t>(1u << oct);
                node.valid_mask |= bit;
                if (children_are_leaves) {
                    node.leaf_mask |= bit;
                    model.attributes.push_back(colour(k.x, k.y, k.z));
                } else {
                    next.push_back(k);
                    model.nodes.emplace_back();
                }
            }
            node.child_base = model.nodes.size() > first_child ? first_child : 0;
            node.attr_base = model.attributes.size() > first_attr ? first_attr : 0;
            model.nodes[level_first + i] = node;
        }
        level_first += static_cast<std::uint32_t>(level_cubes.size());
        level_cubes.swap(next);
    }
    return model;
}

} // namespace voxanim::detail
