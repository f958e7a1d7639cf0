// SVO node addressing, dense-grid build, validation and the .svo stream.
//
// node_child: popcount-rank rule of reference proj/src/svo.cpp:21-39.
// build_from_grid: layout of svo.cpp:80-132 (via bfs_builder.hpp).
// validate/stats: svo.cpp:134-185. serialize/deserialize: svo.cpp:205-291
// (same byte stream, same SvoFormatErrorCode per corruption class).
#include "voxanim/svo.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <fstream>
#include <iterator>

#include "bfs_builder.hpp"

namespace voxanim {

namespace {

constexpr std::uint32_t kDepthLimit = 16;
constexpr std::size_t kHeader = 20, kNodeRec = 12, kAttrRec = 4;
constexpr std::uint32_t kStreamVersion = 1;
constexpr std::uint8_t kMagic[4] = {'S', 'V', 'O', 'A'};

unsigned rank_of(std::uint8_t mask, unsigned octant) {
    return static_cast<unsigned>(std::popcount(static_cast<unsigned>(mask) & ((1u << octant) - 1u)));
}

std::uint8_t internal_mask(const SvoNode& n) { return static_cast<std::uint8_t>(n.valid_mask & ~n.leaf_mask); }
std::uint8_t leaf_children(const SvoNode& n) { return static_cast<std::uint8_t>(n.valid_mask & n.leaf_mask); }

void emit_u32(std::vector<std::uint8_t>& out, std::uint32_t v) {
    for (int s = 0; s < 32; s += 8) out.push_back(static_cast<std::uint8_t>(v >> s));
}

std::uint32_t read_u32(const std::uint8_t* p) {
    return std::uint32_t{p[0]} | (std::uint32_t{p[1]} << 8) | (std::uint32_t{p[2]} << 16) | (std::uint32_t{p[3]} << 24);
}

} // namespace

ChildRef node_child(const SvoModel& model, std::uint32_t node_index, unsigned octant) {
    const SvoNode& n = model.nodes[node_index];
    const unsigned bit = 1u << octant;
    if ((n.valid_mask & bit) == 0) return {};
    if (n.leaf_mask & bit) return {ChildRef::Kind::Leaf, n.attr_base + rank_of(leaf_children(n), octant)};
    return {ChildRef::Kind::Node, n.child_base + rank_of(internal_mask(n), octant)};
}

SvoModel build_from_grid(const VoxelGrid& grid, std::uint32_t depth) {
    if (depth < 1 || depth > kDepthLimit)
        throw ValidationError("octree depth must be in [1, 16], got " + std::to_string(depth));
    if (grid.resolution() != (1u << depth))
        throw ValidationError("grid resolution " + std::to_string(grid.resolution()) +
                              " does not match 2^depth = " + std::to_string(1u << depth));
    // Occupancy pyramid: pyr[L] holds one byte per cube of the 2^L lattice
    // (L < depth); level `depth` is the grid itself.
    std::vector<std::vector<std::uint8_t>> pyr(depth);
    for (int L = static_cast<int>(depth) - 1; L >= 0; --L) {
        const std::uint32_t n = 1u << L;
        auto& cur = pyr[static_cast<std::size_t>(L)];
        cur.assign(std::size_t{n} * n * n, 0);
        for (std::uint32_t x = 0; x < n; ++x)
            for (std::uint32_t y = 0; y < n; ++y)
                for (std::uint32_t z = 0; z < n; ++z) {
                    bool any = false;
                    for (unsigned o = 0; o < 8 && !any; ++o) {
                        const std::uint32_t cx = 2 * x + ((o >> 2) & 1u), cy = 2 * y + ((o >> 1) & 1u),
                                            cz = 2 * z + (o & 1u);
                        if (static_cast<std::uint32_t>(L) + 1 == depth) {
                            any = grid.is_set(cx, cy, cz);
                        } else {
                            const std::uint32_t m = 2 * n;
                            any = pyr[static_cast<std::size_t>(L) + 1][(std::size_t{cx} * m + cy) * m + cz] != 0;
                        }
                    }
                    cur[(std::size_t{x} * n + y) * n + z] = any ? 1 : 0;
                }
    }
    const auto occupied = [&](std::uint32_t L, std::uint32_t x, std::uint32_t y, std::uint32_t z) {
        if (L == depth) return grid.is_set(x, y, z);
        const std::size_t n = std::size_t{1} << L;
        return pyr[L][(x * n + y) * n + z] != 0;
    };
    return detail::build_breadth_first(depth, occupied,
                                       [&](std::uint32_t x, std::uint32_t y, std::uint32_t z) {
                                           return grid.color_at(x, y, z);
                                       });
}

SvoValidationReport validate(const SvoModel& model) {
    SvoValidationReport rep;
    auto flag = [&](std::uint32_t i, const char* what) { rep.violations.push_back({i, what}); };
    if (model.depth < 1 || model.depth > kDepthLimit) flag(0, "depth out of range [1, 16]");
    if (model.nodes.empty()) {
        flag(0, "model has no root node");
        return rep;
    }
    const std::uint64_t nn = model.nodes.size(), na = model.attributes.size();
    for (std::uint32_t i = 0; i < nn; ++i) {
        const SvoNode& n = model.nodes[i];
        if (n.leaf_mask & ~n.valid_mask) flag(i, "leaf not valid: leaf_mask has bits outside valid_mask");
        const unsigned kids = std::popcount(static_cast<unsigned>(internal_mask(n)));
        const unsigned leaves = std::popcount(static_cast<unsigned>(leaf_children(n)));
        if (kids > 0) {
            if (std::uint64_t{n.child_base} + kids > nn)
                flag(i, "child_base out of range");
            else if (n.child_base <= i)
                flag(i, "children do not follow parent (child_base <= node index)");
        }
        if (leaves > 0 && std::uint64_t{n.attr_base} + leaves > na) flag(i, "attr_base out of range");
    }
    return rep;
}

SvoStats stats(const SvoModel& model) {
    SvoStats s;
    s.node_count = model.nodes.size();
    s.depth = model.depth;
    for (const SvoNode& n : model.nodes) s.leaf_count += std::popcount(static_cast<unsigned>(leaf_children(n)));
    s.byte_size = kHeader + kNodeRec * s.node_count + kAttrRec * model.attributes.size();
    s.fill_ratio = static_cast<double>(s.leaf_count) / std::ldexp(1.0, static_cast<int>(3 * model.depth));
    return s;
}

std::vector<std::uint8_t> serialize(const SvoModel& model) {
    std::vector<std::uint8_t> out;
    out.reserve(kHeader + kNodeRec * model.nodes.size() + kAttrRec * model.attributes.size());
    out.insert(out.end(), std::begin(kMagic), std::end(kMagic));
    emit_u32(out, kStreamVersion);
    emit_u32(out, model.depth);
    emit_u32(out, static_cast<std::uint32_t>(model.nodes.size()));
    emit_u32(out, static_cast<std::uint32_t>(model.attributes.size()));
    for (const SvoNode& n : model.nodes) {
        emit_u32(out, n.child_base);
        emit_u32(out, n.attr_base);
        out.insert(out.end(), {n.valid_mask, n.leaf_mask, std::uint8_t{0}, std::uint8_t{0}});
    }
    for (const VoxelAttribute& a : model.attributes) out.insert(out.end(), {a.r, a.g, a.b, a.a});
    return out;
}

SvoModel deserialize(std::span<const std::uint8_t> bytes) {
    using E = SvoFormatErrorCode;
    if (bytes.size() < kHeader) throw SvoFormatError(E::Truncated, "svo: truncated header");
    if (!std::equal(std::begin(kMagic), std::end(kMagic), bytes.begin()))
        throw SvoFormatError(E::BadMagic, "svo: bad magic, not an SVOA file");
    const std::uint8_t* p = bytes.data();
    if (const std::uint32_t v = read_u32(p + 4); v != kStreamVersion)
        throw SvoFormatError(E::BadVersion, "svo: unsupported version " + std::to_string(v));
    const std::uint32_t depth = read_u32(p + 8), nn = read_u32(p + 12), na = read_u32(p + 16);
    if (depth < 1 || depth > kDepthLimit || nn == 0)
        throw SvoFormatError(E::BadHeader, "svo: bad header (depth or node count out of range)");
    const std::size_t want = kHeader + kNodeRec * std::size_t{nn} + kAttrRec * std::size_t{na};
    if (bytes.size() < want) throw SvoFormatError(E::Truncated, "svo: truncated payload");
    if (bytes.size() > want) throw SvoFormatError(E::TrailingData, "svo: trailing bytes after payload");

    SvoModel m;
    m.depth = depth;
    m.nodes.resize(nn);
    m.attributes.resize(na);
    const std::uint8_t* q = p + kHeader;
    for (std::uint32_t i = 0; i < nn; ++i, q += kNodeRec) {
        SvoNode& n = m.nodes[i];
        n = {read_u32(q), read_u32(q + 4), q[8], q[9]};
        const unsigned kids = std::popcount(static_cast<unsigned>(internal_mask(n)));
        const unsigned leaves = std::popcount(static_cast<unsigned>(leaf_children(n)));
        if (kids > 0 && std::uint64_t{n.child_base} + kids > nn)
            throw SvoFormatError(E::NodeIndexOutOfRange, "svo: node " + std::to_string(i) + " child_base out of range");
        if (leaves > 0 && std::uint64_t{n.attr_base} + leaves > na)
            throw SvoFormatError(E::AttrIndexOutOfRange, "svo: node " + std::to_string(i) + " attr_base out of range");
    }
    for (std::uint32_t i = 0; i < na; ++i, q += kAttrRec) m.attributes[i] = {q[0], q[1], q[2], q[3]};
    return m;
}

void save_svo(const std::filesystem::path& path, const SvoModel& model) {
    const auto bytes = serialize(model);
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw IoError("cannot open for writing: " + path.string());
    f.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!f) throw IoError("short write: " + path.string());
}

SvoModel load_svo(const std::filesystem::path& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError("cannot open: " + path.string());
    const std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    return deserialize(bytes);
}

void for_each_leaf(const SvoModel& model,
                   const std::function<void(std::uint32_t, std::uint32_t, std::uint32_t, const VoxelAttribute&)>& fn) {
    if (model.nodes.empty()) return;
    // Depth-first, octant 0 first; leaves above full depth are scaled up.
    const auto walk = [&](const auto& self, std::uint32_t node, std::uint32_t x, std::uint32_t y, std::uint32_t z,
                          std::uint32_t level) -> void {
        for (unsigned oct = 0; oct < 8; ++oct) {
            const ChildRef ref = node_child(model, node, oct);
            if (ref.absent()) continue;
            const std::uint32_t cx = (x << 1) | ((oct >> 2) & 1u), cy = (y << 1) | ((oct >> 1) & 1u),
                                cz = (z << 1) | (oct & 1u);
            if (ref.is_node()) {
                self(self, ref.index, cx, cy, cz, level + 1);
            } else {
                const std::uint32_t sh = model.depth - level - 1;
                fn(cx << sh, cy << sh, cz << sh, model.attributes[ref.index]);
            }
        }
    };
    walk(walk, 0, 0, 0, 0, 0);
}

} // namespace voxanim
