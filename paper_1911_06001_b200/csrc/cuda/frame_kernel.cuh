// The frame kernel: one persistent grid renders a whole frame.
//
// Work distribution: each warp fetches 8x4-pixel tiles from a global atomic
// counter (lane 0 atomicAdd, __shfl_sync broadcast) and walks them until the
// rank's tiles are exhausted; tiles are enumerated super-tile-major so
// neighbouring warps trace neighbouring pixels (coherent node fetches), and
// 64x64 super-tiles are dealt round-robin over ranks for the multi-GPU split.
//
// Per pixel (reference shade_pixel, renderer.cpp:143-214, minus threads):
//   primary ray -> sphere pass over all instances -> [hit-buffer reuse]
//   -> candidates in (t_center, id) order by successive minimum
//   -> trace: skip when best.t < t_boundary, traverse, keep nearest (t, id)
//   -> shade -> RGBA8 store (+ optional AOV / hit-buffer record).
#pragma once

#include "vxa_device.cuh"

namespace vxa {

enum : uint32_t { kMiss = 0, kSingle = 1, kMulti = 2 };

template <typename Real> struct Best {
    bool have;
    Real t;
    int32_t id;
    uint32_t inst;
    TravHit<Real> hit;
    Real normal[3];
};

template <typename Real> struct SphereRes {
    bool hit;
    Real tc, tb;
};

// Bounding-sphere test (renderer.cpp:25-43).
template <typename Real>
__device__ __forceinline__ SphereRes<Real> sphere_test(const DevInstance<Real>& in, const Real d[3]) {
    SphereRes<Real> s;
    if constexpr (sizeof(Real) == 8) {
        // Reference order: t_c = l.d ; d2 = |l|^2 - t_c^2 ; miss iff d2 >= r2 or t_c + r < 0.
        s.tc = in.L[0] * d[0] + in.L[1] * d[1] + in.L[2] * d[2];
        const Real d2 = in.L2 - s.tc * s.tc;
        s.hit = !(d2 >= in.r2) && !(s.tc + in.r < Real(0));
        Real tb = s.tc - sqrt(in.r2 - d2);
        s.tb = tb < Real(0) ? Real(0) : tb;
    } else {
        // FP32: perpendicular form (no |l|^2 - t_c^2 cancellation) and a
        // conservative margin, so rounding can only add candidates or delay a
        // skip; either way the nearest (t, id) result is unchanged.
        s.tc = in.L[0] * d[0] + in.L[1] * d[1] + in.L[2] * d[2];
        const float px = in.L[0] - s.tc * d[0], py = in.L[1] - s.tc * d[1], pz = in.L[2] - s.tc * d[2];
        const float d2 = px * px + py * py + pz * pz;
        const float slack = 1e-5f * in.r2 + 1e-12f;
        s.hit = (d2 < in.r2 + slack) && (s.tc + in.r * 1.00001f >= 0.0f);
        const float tb = s.tc - sqrtf(fmaxf(in.r2 - d2, 0.0f)) - 1e-5f * (fabsf(s.tc) + in.r);
        s.tb = fmaxf(tb, 0.0f);
    }
    return s;
}

// Local direction of instance i for the pixel's camera-space direction.
template <typename Real>
__device__ __forceinline__ void local_dir(const DevInstance<Real>& in, const Real dw[3], const Real dc[3], Real rn,
                                          Real out[3]) {
    if constexpr (sizeof(Real) == 8) {
        // d' = R^T d  (math.hpp:221-224, Mat3*Vec3 row order)
        for (int k = 0; k < 3; ++k) out[k] = in.M[3 * k] * dw[0] + in.M[3 * k + 1] * dw[1] + in.M[3 * k + 2] * dw[2];
    } else {
        // d' = (R^T C) d_cam / |d_cam|
        for (int k = 0; k < 3; ++k)
            out[k] = (in.M[3 * k] * dc[0] + in.M[3 * k + 1] * dc[1] + in.M[3 * k + 2] * dc[2]) * rn;
    }
}

template <typename Real, bool kAov, bool kHbo>
__device__ __forceinline__ void trace_candidate(const FrameParams<Real>& p, uint32_t i, const Real dw[3],
                                                const Real dc[3], Real rn, Best<Real>& best, uint32_t& traversals,
                                                uint32_t& fetches) {
    const DevInstance<Real>& in = p.inst[i];
    if (!in.valid_model) return;
    LocalRay<Real> lr;
    local_dir(in, dw, dc, rn, lr.d);
    setup_root(lr, in.A_lo, in.A_hi, in.zflags, in.zbits);
    ++traversals;
    TravHit<Real> h;
    NoLog nolog;
    const bool hit = traverse_model(in.model, lr, h, nolog);
    fetches += h.fetches;
    if (!hit) return;
    if (!best.have || h.t < best.t || (h.t == best.t && in.id < best.id)) {
        best.have = true;
        best.t = h.t;
        best.id = in.id;
        best.inst = i;
        best.hit = h;
        // world normal = R n_local, n_local = sign e_axis opposing the unmirrored local d
        const int a = static_cast<int>(h.axis);
        const Real sgn = lr.d[a] > Real(0) ? Real(-1) : Real(1);
        Real nl[3] = {Real(0), Real(0), Real(0)};
        nl[a] = sgn;
        for (int k = 0; k < 3; ++k) best.normal[k] = in.R[3 * k] * nl[0] + in.R[3 * k + 1] * nl[1] + in.R[3 * k + 2] * nl[2];
    }
}

// Shade (renderer.cpp:102-113): ambient 0.2 + 0.8 headlight Lambert,
// round half away from zero.
template <typename Real>
__device__ __forceinline__ uint32_t shade_rgba(uint32_t color, const Real n[3], const Real dw[3]) {
    Real facing = n[0] * (-dw[0]) + n[1] * (-dw[1]) + n[2] * (-dw[2]);
    facing = Real(0) < facing ? facing : Real(0);
    const Real f = Real(0.2) + Real(0.8) * facing;
    uint32_t out = 0xff000000u;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const Real ch = static_cast<Real>((color >> (8 * c)) & 0xffu);
        uint32_t v;
        if constexpr (sizeof(Real) == 8)
            v = static_cast<uint32_t>(llround(ch * f));
        else
            v = static_cast<uint32_t>(roundf(ch * f));
        out |= (v & 0xffu) << (8 * c);
    }
    return out;
}

template <typename Real, bool kAov, bool kHbo>
__global__ void __launch_bounds__(128) frame_kernel(const __grid_constant__ FrameParams<Real> p) {
    const uint32_t lane = threadIdx.x & 31u;
    unsigned long long n_rays = 0, n_sph = 0, n_trav = 0, n_reuse = 0, n_fetch = 0, n_leaf = 0;
    const uint32_t n = p.n_inst;

    while (true) {
        uint32_t tile = 0;
        if (lane == 0) tile = atomicAdd(p.tile_counter, 1u);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= p.n_tiles) break;
        const uint32_t st = tile / kTilesPerSuper, wt = tile % kTilesPerSuper;
        const uint32_t s = st * static_cast<uint32_t>(p.world) + static_cast<uint32_t>(p.rank);
        const int px = static_cast<int>((s % p.n_super_x) * kSuper + (wt % (kSuper / kTileW)) * kTileW + (lane % kTileW));
        const int py = static_cast<int>((s / p.n_super_x) * kSuper + (wt / (kSuper / kTileW)) * kTileH + (lane / kTileW));
        if (px >= p.width || py >= p.height) continue;
        const size_t pix = static_cast<size_t>(py) * static_cast<size_t>(p.width) + static_cast<size_t>(px);

        // ---- primary ray (renderer.cpp:11-23)
        Real dw[3], dc[3], rn;
        if constexpr (sizeof(Real) == 8) {
            const double ndc_x = (px + 0.5) / p.width * 2.0 - 1.0;
            const double ndc_y = 1.0 - (py + 0.5) / p.height * 2.0;
            dc[0] = ndc_x * p.tan_half * p.aspect;
            dc[1] = ndc_y * p.tan_half;
            dc[2] = -1.0;
            Real w[3];
            for (int k = 0; k < 3; ++k) w[k] = p.C[3 * k] * dc[0] + p.C[3 * k + 1] * dc[1] + p.C[3 * k + 2] * dc[2];
            const double len = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
            for (int k = 0; k < 3; ++k) dw[k] = w[k] / len;
            rn = 1.0;
        } else {
            const float ndc_x = fmaf(static_cast<float>(px) + 0.5f, p.inv_w2, -1.0f);
            const float ndc_y = fmaf(-(static_cast<float>(py) + 0.5f), p.inv_h2, 1.0f);
            dc[0] = ndc_x * p.sx;
            dc[1] = ndc_y * p.sy;
            dc[2] = -1.0f;
            rn = rsqrtf(fmaf(dc[0], dc[0], fmaf(dc[1], dc[1], 1.0f)));
            for (int k = 0; k < 3; ++k)
                dw[k] = (p.C[3 * k] * dc[0] + p.C[3 * k + 1] * dc[1] + p.C[3 * k + 2] * dc[2]) * rn;
        }
        ++n_rays;

        // ---- sphere pass: count hits, remember the single hit (HBO rule)
        uint32_t n_hits = 0, only = 0;
        if (p.sphere_pass) {
            n_sph += n;
            for (uint32_t i = 0; i < n; ++i) {
                if (sphere_test(p.inst[i], dw).hit) {
                    if (n_hits == 0) only = i;
                    ++n_hits;
                }
            }
        }

        Best<Real> best;
        best.have = false;
        best.t = Real(0);
        best.id = -1;
        best.inst = 0;
        uint32_t traversals = 0, fetches = 0, kind = kMiss;
        bool reused = false;
        bool single_trace = false;
        HitRec prev;
        if constexpr (kHbo) {
            prev = reinterpret_cast<const HitRec*>(p.hbo)[pix];
            if (!p.camera_dirty && n_hits == 1) {
                const DevInstance<Real>& o = p.inst[only];
                if (prev.kind == kSingle && prev.object_id == o.id && !o.dirty) {
                    reused = true;
                } else {
                    single_trace = true; // "trace just this SVO"
                }
            }
        }

        if (!reused) {
            uint32_t n_cand = 0;
            if (single_trace) {
                n_cand = 1;
                trace_candidate<Real, kAov, kHbo>(p, only, dw, dc, rn, best, traversals, fetches);
            } else if (p.sorting) {
                n_cand = p.culling ? n_hits : n;
                // successive minimum over (t_center, index); index order == id order
                Real last_tc = -pos_inf<Real>();
                int last_i = -1;
                while (true) {
                    int k = -1;
                    Real k_tc = Real(0), k_tb = Real(0);
                    for (uint32_t i = 0; i < n; ++i) {
                        const SphereRes<Real> sr = sphere_test(p.inst[i], dw);
                        if (p.culling && !sr.hit) continue;
                        const bool after = sr.tc > last_tc || (sr.tc == last_tc && static_cast<int>(i) > last_i);
                        if (!after) continue;
                        if (k < 0 || sr.tc < k_tc) {
                            k = static_cast<int>(i);
                            k_tc = sr.tc;
                            k_tb = sr.hit ? sr.tb : Real(0);
                        }
                    }
                    if (k < 0) break;
                    last_tc = k_tc;
                    last_i = k;
                    if (best.have && best.t < k_tb) continue; // skip, do not break (renderer.cpp:70-72)
                    trace_candidate<Real, kAov, kHbo>(p, static_cast<uint32_t>(k), dw, dc, rn, best, traversals, fetches);
                }
            } else {
                // id order, zero boundaries: every candidate is traversed
                for (uint32_t i = 0; i < n; ++i) {
                    if (p.culling && !sphere_test(p.inst[i], dw).hit) continue;
                    ++n_cand;
                    trace_candidate<Real, kAov, kHbo>(p, i, dw, dc, rn, best, traversals, fetches);
                }
            }
            if (best.have) kind = n_cand > 1 ? kMulti : kSingle;
            if constexpr (kHbo) {
                if (!p.camera_dirty && p.culling && n_hits == 0) reused = true; // trivial reuse of a miss
            }
        }
        n_trav += traversals;
        n_fetch += fetches;
        if (reused) ++n_reuse;

        // ---- shade + store
        uint32_t rgba;
        HitRec rec;
        if constexpr (kHbo) {
            if (reused && n_hits == 1) {
                rec = prev;
            } else {
                rec.color = best.have ? __ldg(p.inst[best.inst].model.attrs + best.hit.attr) : 0xff000000u;
                rec.pad0 = 0;
                for (int k = 0; k < 3; ++k) rec.normal[k] = best.have ? static_cast<double>(best.normal[k]) : 0.0;
                rec.t = best.have ? static_cast<double>(best.t) : 0.0;
                rec.object_id = best.have ? best.id : -1;
                rec.kind = static_cast<uint8_t>(kind);
                rec.pad1[0] = rec.pad1[1] = rec.pad1[2] = 0;
            }
            if (rec.kind == kMiss) {
                rgba = p.background;
            } else {
                const Real nrm[3] = {static_cast<Real>(rec.normal[0]), static_cast<Real>(rec.normal[1]),
                                     static_cast<Real>(rec.normal[2])};
                rgba = shade_rgba(rec.color, nrm, dw);
            }
            reinterpret_cast<HitRec*>(p.hbo)[pix] = rec;
        } else {
            if (best.have) {
                const uint32_t color = __ldg(p.inst[best.inst].model.attrs + best.hit.attr);
                rgba = shade_rgba(color, best.normal, dw);
            } else {
                rgba = p.background;
            }
        }
        if (best.have) ++n_leaf;
        p.fb[pix] = rgba;

        if constexpr (kAov) {
            PixelAov a;
            a.t = best.have ? static_cast<double>(best.t) : 0.0;
            a.object_id = best.have ? best.id : (kHbo && reused && n_hits == 1 ? -2 : -1);
            a.node_index = best.have ? best.hit.parent : 0u;
            a.attr_index = best.have ? best.hit.attr : 0u;
            if (best.have)
                path_to_voxel(best.hit.path, best.hit.level, a.voxel);
            else
                a.voxel[0] = a.voxel[1] = a.voxel[2] = 0;
            a.level = static_cast<uint8_t>(best.have ? best.hit.level : 0);
            a.kind = static_cast<uint8_t>(kind);
            a.traversals = static_cast<uint16_t>(traversals);
            a.node_fetches = fetches;
            reinterpret_cast<PixelAov*>(p.aov)[pix] = a;
        }
    }

    // warp-aggregated counters (rays, sphere tests, traversals, reuse, fetches, leaf hits)
    unsigned long long vals[6] = {n_rays, n_sph, n_trav, n_reuse, n_fetch, n_leaf};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        unsigned long long v = vals[k];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        if (lane == 0 && v) atomicAdd(p.counters + k, v);
    }
}

} // namespace vxa
