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
    Real A_lo[3], A_hi[3], h2[3];
    uint32_t zb[3], zf = 0;
    Real d[3];
    for (int a = 0; a < 3; ++a) {
        const double o = in.origin[a], h = in.half_extent[a];
        A_lo[a] = static_cast<Real>(-h - o);
        A_hi[a] = static_cast<Real>(h - o);
        h2[a] = static_cast<Real>(2.0 * h);
        zb[a] = zero_dir_bits(o, h);
        if (-h > o) zf |= 1u << a;
        if (h > o) zf |= 1u << (3 + a);
        d[a] = static_cast<Real>(in.direction[a]);
    }
    TraverseRayOut o{};
    bool hit;
    uint32_t axis = 0, attr = 0, parent = 0, level = 0;
    unsigned long long path = 0;
    double t = 0, te = 0, tx = 0;
    if constexpr (sizeof(Real) == 8) {
        LocalRay<Real> r;
        for (int a = 0; a < 3; ++a) r.d[a] = d[a];
        setup_root(r, A_lo, A_hi, zf, zb);
        BufferLog lg{log != nullptr ? log + static_cast<size_t>(i) * cap : nullptr, cap, 0};
        TravHit<Real> h;
        hit = traverse_model(m, r, h, lg);
        o.node_fetches = h.fetches;
        o.log_total = lg.n;
        o.log_count = lg.n < cap ? lg.n : cap;
        if (hit) t = h.t, te = h.t_enter_root, tx = h.t_exit_root, axis = h.axis, attr = h.attr, parent = h.parent,
                 level = h.level, path = h.path;
    } else {
        FastRay r;
        hit = false;
        o.node_fetches = 0;
        float U_lo[3], U_hi[3], Ur_lo[3], Ur_hi[3];
        for (int a = 0; a < 3; ++a) {
            const double o = in.origin[a], h = in.half_extent[a];
            const double ulo = (-h - o) / (2.0 * h), uhi = (h - o) / (2.0 * h);
            U_lo[a] = static_cast<float>(ulo);
            U_hi[a] = static_cast<float>(uhi);
            Ur_lo[a] = static_cast<float>(ulo - static_cast<double>(U_lo[a]));
            Ur_hi[a] = static_cast<float>(uhi - static_cast<double>(U_hi[a]));
        }
        LocalStack lstack;
        if (fast_setup(r, d, U_lo, U_hi, Ur_lo, Ur_hi, h2, zf, zb)) {
            FastHit h;
            // the frame kernel's dispatch: position-space loop unless a direction component is zero
            if (VXA_POSLOOP && !r.zero)
                hit = traverse_pos<true>(WideNodes{m.words, m.side}, static_cast<int>(m.depth), r, h, lstack);
            else
                hit = traverse_fast<true>(WideNodes{m.words, m.side}, static_cast<int>(m.depth), r, h, lstack);
            o.node_fetches = h.fetches;
            if (hit) {
                t = h.t, axis = h.axis, attr = h.attr, parent = h.parent, level = h.level;
                // leaf path from the voxel coordinates (leaf_path_to_voxel inverted)
                for (uint32_t l = 0; l < level; ++l) {
                    const uint32_t sh = level - 1 - l;
                    const uint32_t oc = (((h.vox[0] >> sh) & 1u) << 2) | (((h.vox[1] >> sh) & 1u) << 1) | ((h.vox[2] >> sh) & 1u);
                    path |= static_cast<unsigned long long>(oc) << (4 * l);
                }
            }
        }
    }
    o.hit = hit ? 1 : 0;
    if (hit) {
        o.t_hit = t;
        o.t_enter = te;
        o.t_exit = tx;
        o.normal_local[axis] = in.direction[axis] > 0.0 ? -1.0 : 1.0;
        const uint32_t rgba = __ldg(m.attrs + attr);
        for (int k = 0; k < 4; ++k) o.attribute[k] = static_cast<uint8_t>(rgba >> (8 * k));
        o.attr_index = attr;
        o.node_index = parent;
        o.path_len = static_cast<uint8_t>(level);
        for (int l = 0; l < 16; ++l) o.leaf_path[l] = static_cast<uint8_t>((path >> (4 * l)) & 0xfu);
    }
    out[i] = o;
}

} // namespace vxa
