// Production frame kernel (FP32, bounding-sphere culling on, no hit buffer):
// persistent warps with per-lane ray replacement.
//
// The straightforward kernel (frame_kernel.cuh) runs a warp over one 8x4
// tile and waits for its slowest pixel: rays that miss every sphere, hit one
// instance, or walk a long grazing path all share a warp, so only ~13 of 32
// lanes are active on average (ncu smsp__thread_inst_executed_per_inst_executed).
// Here every lane owns one pixel at a time and keeps its whole state in
// registers (traversal) and shared memory (node stack); when enough lanes
// have finished their pixel, the warp refills them from its tile pool
// (Aila & Laine's persistent "while-while" with dynamic ray fetch), building
// the tile's cone-culled instance list whenever it opens a new 8x4 tile.
//
// Each pixel follows the reference shade_pixel without a hit buffer
// (renderer.cpp:143-214): sphere pass, candidates in (t_center, id) order (id
// order when sorting is off), skip-not-break on t_boundary, nearest (t, id).
// A pixel whose tile list overflows (> 64 instances) or whose ray meets more
// than kQueue spheres is appended to an overflow list that the generic kernel
// finishes in a second launch, with the same FP32 arithmetic.
#pragma once

#include "frame_kernel.cuh"

namespace vxa {

#ifndef VXA_FAST_MIN_BLOCKS
#define VXA_FAST_MIN_BLOCKS 6
#endif

constexpr uint32_t kQueue = 8; // candidates per pixel kept in the lane's queue (4 x 16 bits per u64)

struct LaneTrav {
    FastRay r;
    DevModel m;
    float c[3];
    float sz;
    float t0[3], tm[3], t1[3];
    uint2 fw;
    uint32_t fcur, fidx, fetches;
    int level, depth;
};

// One step of traverse_fast (vxa_device.cuh): returns 0 while running,
// 1 on a hit (h filled), 2 when the ray leaves the root.
template <bool kTrackIdx>
__device__ __forceinline__ int trav_step(LaneTrav& s, FastHit& h, uint2* __restrict__ stack, uint32_t* sidx) {
    if (s.fcur == kExit) {
        if (s.level == 0) return 2;
        --s.level;
        s.fw = stack[s.level * kBlock];
        s.fcur = (s.fw.x >> 24) & 0xfu;
        s.fw.x &= 0x00ffffffu;
        if constexpr (kTrackIdx) s.fidx = sidx[s.level];
        s.sz = 2.0f * s.sz;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float cp = floorf(0.5f * s.c[a]);
            const bool upper = s.c[a] != 2.0f * cp;
            s.c[a] = cp;
            if (upper) {
                s.tm[a] = s.t0[a];
                s.t0[a] = plane_t(cp, s.sz, s.r.A[a], s.r.Ar[a], s.r.inv[a]);
            } else {
                s.tm[a] = s.t1[a];
                s.t1[a] = plane_t(cp + 1.0f, s.sz, s.r.A[a], s.r.Ar[a], s.r.inv[a]);
            }
        }
        if (s.r.zero) fix_zero_axes(s.r, s.level, s.t0, s.tm, s.t1);
        return 0;
    }
    const uint32_t q = s.fcur;
    float c0[3], c1[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const bool up = (q & axis_bit(a)) != 0;
        c0[a] = up ? s.tm[a] : s.t0[a];
        c1[a] = up ? s.t1[a] : s.tm[a];
    }
    s.fcur = next_child(c1, q);
    int entry = 0;
    float t_enter = c0[0];
    if (c0[1] > t_enter) {
        entry = 1;
        t_enter = c0[1];
    }
    if (c0[2] > t_enter) {
        entry = 2;
        t_enter = c0[2];
    }
    const float t_exit = fminf(fminf(c1[0], c1[1]), c1[2]);
    if (!(t_enter < t_exit) || t_exit < 0.0f) return 0;
    const uint32_t oct = q ^ s.r.mirror;
    const uint32_t bit = 1u << oct;
    const uint32_t valid = s.fw.x & 0xffu;
    const uint32_t leafm = (s.fw.x >> 8) & 0xffu;
    if (!(valid & bit)) return 0;
    if (leafm & bit) {
        const uint32_t abase = (s.fw.x & kMixed) ? __ldg(s.m.side + s.fw.y) : s.fw.y;
        h.attr = abase + popc8_below(valid & leafm, bit);
        h.t = fmaxf(t_enter, 0.0f);
        h.parent = s.fidx;
        h.level = static_cast<uint32_t>(s.level + 1);
        h.axis = static_cast<uint32_t>(entry);
        h.fetches = s.fetches;
        const uint32_t top = (2u << s.level) - 1u;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const uint32_t v = 2u * static_cast<uint32_t>(s.c[a]) + ((q >> (2 - a)) & 1u);
            h.vox[a] = (s.r.mirror & axis_bit(a)) ? top - v : v;
        }
        return 1;
    }
    if (s.level + 1 >= s.depth) return 0;
    const uint32_t child = s.fw.y + popc8_below(valid & ~leafm, bit);
    stack[s.level * kBlock] = make_uint2(s.fw.x | (s.fcur << 24), s.fw.y);
    if constexpr (kTrackIdx) {
        sidx[s.level] = s.fidx;
        s.fidx = child;
    }
    ++s.level;
    s.fw = load_node(s.m, child);
    ++s.fetches;
    s.sz = 0.5f * s.sz;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        s.c[a] = __fmaf_rn(2.0f, s.c[a], static_cast<float>((q >> (2 - a)) & 1u));
        s.t0[a] = c0[a];
        s.t1[a] = c1[a];
        s.tm[a] = plane_t(__fmaf_rn(2.0f, s.c[a], 1.0f), 0.5f * s.sz, s.r.A[a], s.r.Ar[a], s.r.inv[a]);
    }
    if (s.r.zero) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
            if (s.r.zero & axis_bit(a)) s.tm[a] = zero_mid(s.r, a, s.level);
    }
    s.fcur = first_child(s.t0, s.tm);
    return 0;
}

// Root of instance i for the pixel (FP64 local direction rounded once).
// Returns false when the ray misses the instance's box.
__device__ __forceinline__ bool trav_begin(const FrameParams<float>& p, uint32_t i, int px, int py, double rnd,
                                           LaneTrav& s) {
    const DevInstance<float>& in = p.inst[i];
    const double dcx = fma(static_cast<double>(px) + 0.5, p.d_inv_w2, -1.0) * p.d_sx;
    const double dcy = fma(-(static_cast<double>(py) + 0.5), p.d_inv_h2, 1.0) * p.d_sy;
    float d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        d[k] = static_cast<float>((fma(in.Md[3 * k], dcx, in.Md[3 * k + 1] * dcy) - in.Md[3 * k + 2]) * rnd);
    if (!fast_setup(s.r, d, in.U_lo, in.U_hi, in.Ur_lo, in.Ur_hi, in.h2, in.zflags, in.zbits)) return false;
    s.m = in.model;
    s.depth = min(static_cast<int>(in.model.depth), static_cast<int>(kMaxDepth));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        s.c[a] = 0.0f;
        s.t0[a] = plane_t(0.0f, 1.0f, s.r.A[a], s.r.Ar[a], s.r.inv[a]);
        s.t1[a] = plane_t(1.0f, 1.0f, s.r.A[a], s.r.Ar[a], s.r.inv[a]);
        s.tm[a] = plane_t(1.0f, 0.5f, s.r.A[a], s.r.Ar[a], s.r.inv[a]);
    }
    if (s.r.zero) fix_zero_axes(s.r, 0, s.t0, s.tm, s.t1);
    s.sz = 1.0f;
    s.level = 0;
    s.fidx = 0;
    s.fetches = 1;
    s.fw = load_node(s.m, 0);
    s.fcur = first_child(s.t0, s.tm);
    return true;
}

template <bool kAov>
__global__ void __launch_bounds__(kBlock, VXA_FAST_MIN_BLOCKS) frame_kernel_fast(const __grid_constant__ FrameParams<float> p) {
    extern __shared__ uint2 smem_stack[]; // [level][thread]
    __shared__ uint16_t s_list[kWarps][kListCap];
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint2* const stack = smem_stack + threadIdx.x;
    uint16_t* const list = s_list[warp];
    const uint32_t n = p.n_inst;
    uint32_t sidx[kAov ? kMaxDepth : 1];

    // warp-uniform pool state
    uint32_t pool_next = 32, list_n = 0;
    bool list_ok = false, exhausted = false;
    int tx0 = 0, ty0 = 0;

    // lane state
    bool busy = false; // a pixel is in flight (traversing one of its candidates)
    int px = 0, py = 0;
    double rnd = 0.0;
    float dw[3] = {0.0f, 0.0f, 0.0f};
    unsigned long long q0 = 0, q1 = 0; // pending candidates, 16 bits each, front in the low bits
    uint32_t qn = 0, n_cand = 0, traversals = 0, fetches = 0, cur = 0;
    bool have = false, pos_dir = false;
    float best_t = 0.0f;
    int32_t best_id = -1;
    uint32_t best_inst = 0, best_axis = 0, best_attr = 0, best_parent = 0, best_level = 0, best_vox[3] = {0, 0, 0};
    LaneTrav s;
    uint32_t n_trav = 0, n_fetch = 0, n_leaf = 0;

    // Pops candidates until one starts a traversal (skip rule, invalid models,
    // box misses); false when the pixel has no candidate left.
    auto next_traversal = [&]() -> bool {
        while (qn > 0) {
            const uint32_t i = static_cast<uint32_t>(q0 & 0xffffu);
            q0 = (q0 >> 16) | (q1 << 48);
            q1 >>= 16;
            --qn;
            if (p.sorting) {
                const SphereRes<float> sr = sphere_test(p.inst[i], dw);
                if (have && best_t < sr.tb) continue; // skip, do not break (renderer.cpp:70-72)
            }
            if (!p.inst[i].valid_model) continue;
            ++traversals;
            cur = i;
            if (trav_begin(p, i, px, py, rnd, s)) return true;
        }
        return false;
    };

    auto finish_pixel = [&]() {
        const size_t pix = static_cast<size_t>(py) * static_cast<size_t>(p.width) + static_cast<size_t>(px);
        uint32_t rgba = p.background;
        if (have) {
            const DevInstance<float>& in = p.inst[best_inst];
            float nl[3] = {0.0f, 0.0f, 0.0f};
            nl[best_axis] = pos_dir ? -1.0f : 1.0f;
            float nrm[3];
            for (int k = 0; k < 3; ++k) nrm[k] = in.R[3 * k] * nl[0] + in.R[3 * k + 1] * nl[1] + in.R[3 * k + 2] * nl[2];
            rgba = shade_rgba(__ldg(in.model.attrs + best_attr), nrm, dw);
            ++n_leaf;
        }
        p.fb[pix] = rgba;
        n_trav += traversals;
        n_fetch += fetches;
        if constexpr (kAov) {
            PixelAov a;
            a.t = have ? static_cast<double>(best_t) : 0.0;
            a.object_id = have ? best_id : -1;
            a.node_index = have ? best_parent : 0u;
            a.attr_index = have ? best_attr : 0u;
            a.voxel[0] = have ? best_vox[0] : 0u;
            a.voxel[1] = have ? best_vox[1] : 0u;
            a.voxel[2] = have ? best_vox[2] : 0u;
            a.level = static_cast<uint8_t>(have ? best_level : 0u);
            a.kind = static_cast<uint8_t>(have ? (n_cand > 1 ? kMulti : kSingle) : kMiss);
            a.entry_axis = static_cast<uint8_t>(have ? best_axis : 0u);
            a.pad0 = 0;
            a.traversals = traversals;
            a.node_fetches = fetches;
            a.pad1 = 0;
            reinterpret_cast<PixelAov*>(p.aov)[pix] = a;
        }
        busy = false;
    };

    // Starts pixel k of the open tile: ray, sphere pass over the tile list,
    // ordered queue. Pixels it cannot hold go to the overflow list.
    auto start_pixel = [&](uint32_t k) {
        px = tx0 + static_cast<int>(k % kTileW);
        py = ty0 + static_cast<int>(k / kTileW);
        if (px >= p.width || py >= p.height) return;
        const float dcx = fmaf(static_cast<float>(px) + 0.5f, p.inv_w2, -1.0f) * p.sx;
        const float dcy = fmaf(-(static_cast<float>(py) + 0.5f), p.inv_h2, 1.0f) * p.sy;
        const float rn = rsqrtf(fmaf(dcx, dcx, fmaf(dcy, dcy, 1.0f)));
        for (int a = 0; a < 3; ++a) dw[a] = (p.C[3 * a] * dcx + p.C[3 * a + 1] * dcy - p.C[3 * a + 2]) * rn;
        const double ddx = fma(static_cast<double>(px) + 0.5, p.d_inv_w2, -1.0) * p.d_sx;
        const double ddy = fma(-(static_cast<double>(py) + 0.5), p.d_inv_h2, 1.0) * p.d_sy;
        rnd = rsqrt(fma(ddx, ddx, fma(ddy, ddy, 1.0)));
        unsigned long long hitmask = 0;
        if (list_ok)
            for (uint32_t j = 0; j < list_n; ++j)
                if (sphere_test(p.inst[list[j]], dw).hit) hitmask |= 1ull << j;
        const uint32_t hits = __popcll(hitmask);
        if (!list_ok || hits > kQueue) {
            const uint32_t slot = atomicAdd(p.ovf_count, 1u);
            p.ovf_list[slot] = static_cast<uint32_t>(py) * static_cast<uint32_t>(p.width) + static_cast<uint32_t>(px);
            return;
        }
        // queue in (t_center, index) order (index order when sorting is off)
        q0 = q1 = 0;
        qn = 0;
        for (unsigned long long rem = hitmask; rem;) {
            int kb = __ffsll(rem) - 1;
            if (p.sorting) {
                float tcb = sphere_test(p.inst[list[kb]], dw).tc;
                for (unsigned long long it = rem & (rem - 1); it; it &= it - 1) {
                    const int j = __ffsll(it) - 1;
                    const float tc = sphere_test(p.inst[list[j]], dw).tc;
                    if (tc < tcb) kb = j, tcb = tc;
                }
            }
            rem &= ~(1ull << kb);
            const unsigned long long v = static_cast<unsigned long long>(list[kb]) << (16 * (qn & 3u));
            if (qn < 4) q0 |= v; else q1 |= v;
            ++qn;
        }
        n_cand = hits;
        have = false;
        best_t = 0.0f;
        best_id = -1;
        traversals = fetches = 0;
        busy = true;
        if (!next_traversal()) finish_pixel();
    };

    while (true) {
        // ---- refill idle lanes from the warp's tile pool
        uint32_t idle = __ballot_sync(0xffffffffu, !busy);
        while (idle != 0 && !exhausted) {
            if (pool_next == 32) {
                uint32_t tile = 0;
                if (lane == 0) tile = atomicAdd(p.tile_counter, 1u);
                tile = __shfl_sync(0xffffffffu, tile, 0);
                if (tile >= p.n_tiles) {
                    exhausted = true;
                    break;
                }
                const uint32_t st = tile / kTilesPerSuper, wt = tile % kTilesPerSuper;
                const uint32_t sp = st * static_cast<uint32_t>(p.world) + static_cast<uint32_t>(p.rank);
                tx0 = static_cast<int>((sp % p.n_super_x) * kSuper + (wt % (kSuper / kTileW)) * kTileW);
                ty0 = static_cast<int>((sp / p.n_super_x) * kSuper + (wt / (kSuper / kTileW)) * kTileH);
                const TileCone cone = tile_cone(p, tx0, ty0);
                uint32_t cnt = 0;
                for (uint32_t base = 0; base < n; base += 32) {
                    const uint32_t i = base + lane;
                    const bool c = i < n && cone_candidate(p.inst[i], cone);
                    const uint32_t msk = __ballot_sync(0xffffffffu, c);
                    const uint32_t pos = cnt + __popc(msk & lt_mask);
                    if (c && pos < kListCap) list[pos] = static_cast<uint16_t>(i);
                    cnt += __popc(msk);
                }
                __syncwarp();
                list_ok = cnt <= kListCap;
                list_n = list_ok ? cnt : 0;
                pool_next = 0;
            }
            const uint32_t avail = 32u - pool_next;
            const uint32_t take = min(static_cast<uint32_t>(__popc(idle)), avail);
            const uint32_t rank_idle = __popc(idle & lt_mask);
            if (!busy && rank_idle < take) start_pixel(pool_next + rank_idle);
            pool_next += take;
            idle = __ballot_sync(0xffffffffu, !busy);
        }
        if (exhausted && idle == 0xffffffffu) break;

        // ---- trace until a quarter of the warp is idle (all of it once the pool is dry)
        while (true) {
            if (busy) {
                FastHit h;
                const int st = trav_step<kAov>(s, h, stack, sidx);
                if (st != 0) {
                    fetches += s.fetches;
                    if (st == 1) {
                        const int32_t id = p.inst[cur].id;
                        if (!have || h.t < best_t || (h.t == best_t && id < best_id)) {
                            have = true;
                            best_t = h.t;
                            best_id = id;
                            best_inst = cur;
                            best_attr = h.attr;
                            best_axis = h.axis;
                            pos_dir = !(s.r.mirror & axis_bit(static_cast<int>(h.axis))) &&
                                      !(s.r.zero & axis_bit(static_cast<int>(h.axis)));
                            if constexpr (kAov) {
                                best_parent = h.parent;
                                best_level = h.level;
                                best_vox[0] = h.vox[0], best_vox[1] = h.vox[1], best_vox[2] = h.vox[2];
                            }
                        }
                    }
                    if (!next_traversal()) finish_pixel();
                }
            }
            const uint32_t n_idle = __popc(__ballot_sync(0xffffffffu, !busy));
            if (n_idle == 32u || (!exhausted && n_idle >= 8u)) break;
        }
    }

    const uint32_t vals[3] = {n_trav, n_fetch, n_leaf};
    const uint32_t slot[3] = {2, 4, 5}; // traversals, node fetches, leaf hits
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const uint32_t v = __reduce_add_sync(0xffffffffu, vals[k]);
        if (lane == 0 && v) atomicAdd(p.counters + slot[k], static_cast<unsigned long long>(v));
    }
}

} // namespace vxa
