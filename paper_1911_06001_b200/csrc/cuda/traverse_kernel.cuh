// Batched single-ray traversal: the GPU body of voxanim::traverse /
// traverse_debug (reference proj/src/traversal.cpp:249-258). Each thread takes
// one local ray + bounds, derives the root slab exactly as ray_box_params does
// (traversal.cpp:30-61), runs traverse_model and writes a TraversalHit-shaped
// record, optionally logging every visited present child.
#pragma once

#include "vxa_internal.h"

namespace vxa {

struct BufferLog {
    VisitOut* buf;
    uint32_t cap;
    uint32_t n;
    __device__ __forceinline__ void visit(double t, uint32_t level, bool leaf) {
        if (buf != nullptr && n < cap) {
            VisitOut v;
            v.t_enter = t;
            v.level = static_cast<uint8_t>(level);
            v.leaf = leaf ? 1 : 0;
            for (int k = 0; k < 6; ++k) v.pad[k] = 0;
            buf[n] = v;
        }
        ++n;
    }
};

template <typename Real>
__global__ void __launch_bounds__(128) traverse_kernel(DevModel m, const TraverseRayIn* __restrict__ rays, uint32_t n,
                                                       TraverseRayOut* __restrict__ out, VisitOut* log, uint32_t cap) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const TraverseRayIn in = rays[i];
    Real A_lo[3], A_hi[3];
    uint32_t zb[3], zf = 0;
    LocalRay<Real> r;
    for (int a = 0; a < 3; ++a) {
        const double o = in.origin[a], h = in.half_extent[a];
        A_lo[a] = static_cast<Real>(-h - o);
        A_hi[a] = static_cast<Real>(h - o);
        zb[a] = zero_dir_bits(o, h);
        if (-h > o) zf |= 1u << a;
        if (h > o) zf |= 1u << (3 + a);
        r.d[a] = static_cast<Real>(in.direction[a]);
    }
    setup_root(r, A_lo, A_hi, zf, zb);
    BufferLog lg{log != nullptr ? log + static_cast<size_t>(i) * cap : nullptr, cap, 0};
    TravHit<Real> h;
    const bool hit = traverse_model(m, r, h, lg);
    TraverseRayOut o{};
    o.hit = hit ? 1 : 0;
    o.node_fetches = h.fetches;
    o.log_total = lg.n;
    o.log_count = lg.n < cap ? lg.n : cap;
    if (hit) {
        o.t_hit = static_cast<double>(h.t);
        o.t_enter = static_cast<double>(h.t_enter_root);
        o.t_exit = static_cast<double>(h.t_exit_root);
        const int a = static_cast<int>(h.axis);
        o.normal_local[a] = in.direction[a] > 0.0 ? -1.0 : 1.0;
        const uint32_t rgba = __ldg(m.attrs + h.attr);
        for (int k = 0; k < 4; ++k) o.attribute[k] = static_cast<uint8_t>(rgba >> (8 * k));
        o.attr_index = h.attr;
        o.node_index = h.parent;
        o.path_len = static_cast<uint8_t>(h.level);
        for (int l = 0; l < 16; ++l) o.leaf_path[l] = static_cast<uint8_t>((h.path >> (4 * l)) & 0xfu);
    }
    out[i] = o;
}

} // namespace vxa
