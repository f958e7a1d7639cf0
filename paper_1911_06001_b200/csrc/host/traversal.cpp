// Per-ray traversal API.
//
// ray_box_params / first_node / next_node are the small slab and ordering
// helpers of reference proj/src/traversal.cpp:30-103 (mirror mask, +/-inf
// zero-direction convention, x > y > z tie priority). traverse and
// traverse_debug dispatch to the GPU (vxa_traverse, FP64 parity kernel), so
// the per-ray API returns exactly the reference's TraversalHit.
#include "voxanim/traversal.hpp"

#include <algorithm>
#include <limits>

#include "voxanim/gpu.hpp"

namespace voxanim {

namespace {

constexpr double kInfinity = std::numeric_limits<double>::infinity();
constexpr unsigned kBit[3] = {octant_bit_x, octant_bit_y, octant_bit_z};

// Plane parameter for a zero direction component: the ray never reaches a
// plane ahead of it and has already passed one at or behind it.
double never_or_always(double plane, double origin) { return plane > origin ? kInfinity : -kInfinity; }

vxa_local_ray to_abi(const Ray& r, const OctreeBounds& b) {
    return {{r.origin.x, r.origin.y, r.origin.z},
            {r.direction.x, r.direction.y, r.direction.z},
            {b.half_extent.x, b.half_extent.y, b.half_extent.z}};
}

TraversalHit from_abi(const vxa_traverse_hit& h) {
    TraversalHit out;
    out.t_hit = h.t_hit;
    out.t_enter = h.t_enter;
    out.t_exit = h.t_exit;
    out.attribute = {h.attribute[0], h.attribute[1], h.attribute[2], h.attribute[3]};
    out.normal_local = {h.normal_local[0], h.normal_local[1], h.normal_local[2]};
    std::copy(std::begin(h.leaf_path), std::end(h.leaf_path), out.leaf_path.begin());
    out.path_len = h.path_len;
    return out;
}

} // namespace

std::optional<BoxParams> ray_box_params(const Ray& ray, const OctreeBounds& bounds) {
    BoxParams p;
    for (int a = 0; a < 3; ++a) {
        const double h = bounds.half_extent[a];
        double o = ray.origin[a], d = ray.direction[a];
        if (d < 0.0) {
            p.mirror_mask |= static_cast<std::uint8_t>(kBit[a]);
            o = -o;
            d = -d;
        }
        if (d == 0.0) {
            p.t0[a] = never_or_always(-h, o);
            p.t1[a] = never_or_always(h, o);
        } else {
            p.t0[a] = (-h - o) / d;
            p.t1[a] = (h - o) / d;
        }
    }
    const double enter = std::max({p.t0[0], p.t0[1], p.t0[2]});
    const double exit = std::min({p.t1[0], p.t1[1], p.t1[2]});
    if (enter >= exit || exit < 0.0) return std::nullopt;
    return p;
}

unsigned first_node(double tx0, double ty0, double tz0, double txm, double tym, double tzm) {
    double enter = tx0;
    if (ty0 > enter) enter = ty0;
    if (tz0 > enter) enter = tz0;
    return (txm < enter ? octant_bit_x : 0u) | (tym < enter ? octant_bit_y : 0u) | (tzm < enter ? octant_bit_z : 0u);
}

unsigned next_node(double tx1, double ty1, double tz1, unsigned current) {
    unsigned bit = octant_bit_x;
    double lowest = tx1;
    if (ty1 < lowest) {
        bit = octant_bit_y;
        lowest = ty1;
    }
    if (tz1 < lowest) bit = octant_bit_z;
    return (current & bit) ? kTraversalExit : (current | bit);
}

std::optional<TraversalHit> traverse(const SvoModel& model, const Ray& ray_local, const OctreeBounds& bounds) {
    const std::uint32_t handle = gpu::model_handle(model);
    const vxa_local_ray in = to_abi(ray_local, bounds);
    vxa_traverse_hit out{};
    gpu::check(vxa_traverse(gpu::context(), handle, &in, 1, VXA_FP64, &out, nullptr, 0), "vxa_traverse");
    if (!out.hit) return std::nullopt;
    return from_abi(out);
}

std::optional<TraversalHit> traverse_debug(const SvoModel& model, const Ray& ray_local, const OctreeBounds& bounds,
                                           std::vector<TraversalVisit>& log) {
    const std::uint32_t handle = gpu::model_handle(model);
    const vxa_local_ray in = to_abi(ray_local, bounds);
    std::uint32_t cap = 256;
    while (true) {
        std::vector<vxa_visit> buf(cap);
        vxa_traverse_hit out{};
        gpu::check(vxa_traverse(gpu::context(), handle, &in, 1, VXA_FP64, &out, buf.data(), cap), "vxa_traverse");
        if (out.log_total > cap) {
            cap = out.log_total;
            continue;
        }
        for (std::uint32_t i = 0; i < out.log_count; ++i)
            log.push_back({buf[i].t_enter, buf[i].level, buf[i].leaf != 0});
        if (!out.hit) return std::nullopt;
        return from_abi(out);
    }
}

std::array<std::uint32_t, 3> leaf_path_to_voxel(std::span<const std::uint8_t> path) {
    std::array<std::uint32_t, 3> v{0, 0, 0};
    for (const std::uint8_t o : path) {
        v[0] = (v[0] << 1) | ((o >> 2) & 1u);
        v[1] = (v[1] << 1) | ((o >> 1) & 1u);
        v[2] = (v[2] << 1) | (o & 1u);
    }
    return v;
}

} // namespace voxanim
