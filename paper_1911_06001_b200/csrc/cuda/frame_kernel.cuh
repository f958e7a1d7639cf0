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

#ifndef VXA_BLOCK
#define VXA_BLOCK 128
#endif
constexpr int kBlock = VXA_BLOCK;
// Minimum resident blocks per SM requested from ptxas for the FP32 kernel
// (register budget 65536 / (128 * n)); tuned by measurement.
#ifndef VXA_MIN_BLOCKS_F64
#define VXA_MIN_BLOCKS_F64 5 // the FP64 parity kernel: 96 registers (4 blocks at 112 without a cap: -5.6 %; 6 blocks: -3.6 %)
#endif
#ifndef VXA_MIN_BLOCKS
#define VXA_MIN_BLOCKS 8
#endif
// Build variants measured in DESIGN.md §7 (defaults = the measured best):
// VXA_PDL      launch the frame kernel as a programmatic dependent of the culling
//              pre-pass (griddepcontrol) -- no change measured, off;
// VXA_ZERO_SPLIT  a second traversal instantiation for rays with a zero local
//              direction component, so the common loop has no zero conventions.
#ifndef VXA_PDL
#define VXA_PDL 0
#endif
#ifndef VXA_ZERO_SPLIT
#define VXA_ZERO_SPLIT 1
#endif
constexpr int kWarps = kBlock / 32;
constexpr uint32_t kListCap = 64; // per-warp tile candidate list (bit positions of a u64 mask)
// bytes per thread per level (the node-word part's stride; layout 2 keeps the
// entry parameters in a second array of half that stride)
constexpr uint32_t kStackEntry = (VXA_STACK_TEN && VXA_STACK_LAYOUT != 2) ? 16u : 8u;
constexpr uint32_t kStackBytes = VXA_STACK_TEN ? (VXA_STACK_LAYOUT == 2 ? 12u : 16u) : 8u; // per thread per level
// Stack levels a frame needs: a node is saved only when one of its internal
// children is pushed, i.e. at levels <= depth - 2 (VXA_STACK_TRIM; else depth).
// Together with layout 2: 15 KB of stack per block at C4 instead of 22.5 (-1.1 %).
#ifndef VXA_STACK_TRIM
#define VXA_STACK_TRIM 1
#endif
__host__ __device__ inline uint32_t stack_levels(uint32_t max_depth) {
    const uint32_t d = max_depth > 0 ? max_depth : 1u;
    return VXA_STACK_TRIM ? (d > 1 ? d - 1 : 1u) : d;
}
struct BlockStack : SmemStack<kBlock * kStackEntry> {
    uint32_t base_top; // shared address of the staged top node words (VXA_SMEM_TOP)
};

// Super-tile row of super-tile s: s / n_super_x by a multiply-high when the
// host found the magic exact for every super-tile of the frame (vxa_abi.cu).
template <typename Real> __device__ __forceinline__ uint32_t super_row(const FrameParams<Real>& p, uint32_t s) {
    return p.super_x_magic ? __umulhi(s, p.super_x_magic) : s / p.n_super_x;
}

// The nearest hit so far of a pixel: t, instance, attribute, entry axis and
// whether the unmirrored local direction is positive on it (the normal's sign);
// parent / level / voxel for the AOV kernels only.
template <typename Real> struct Best {
    Real t = Real(0);
    bool have_ = false, pos_dir_ = false;
    int32_t id_ = -1;
    uint32_t inst_ = 0, axis_ = 0;
    uint32_t attr = 0, parent = 0, level = 0;
    uint32_t vox[3] = {0, 0, 0};
    __device__ __forceinline__ bool have() const { return have_; }
    __device__ __forceinline__ uint32_t inst() const { return inst_; }
    __device__ __forceinline__ uint32_t axis() const { return axis_; }
    __device__ __forceinline__ bool pos_dir() const { return pos_dir_; }
    __device__ __forceinline__ int32_t id(const FrameParams<Real>&) const { return id_; }
    __device__ __forceinline__ void set(uint32_t inst, int32_t id, uint32_t axis, bool pos_dir) {
        have_ = true, inst_ = inst, id_ = id, axis_ = axis, pos_dir_ = pos_dir;
    }
};

// FP32 kernel: few registers live across the candidate loop (they spill at the
// 64-register cap). Instance, axis, sign and the have-flag share one word; the
// object id is read back from the instance record when needed (exact t ties,
// outputs); t is in the pixel's traversal units (unnormalised camera direction
// u, see camera_dir_f64): t_world = t |u|.
template <> struct Best<float> {
    float t = 0.0f;
    uint32_t key = 0; // bit 31 have | bit 26 pos_dir | bits 24-25 axis | bits 0-23 instance
    uint32_t attr = 0, parent = 0, level = 0;
    uint32_t vox[3] = {0, 0, 0};
    __device__ __forceinline__ bool have() const { return (key >> 31) != 0; }
    __device__ __forceinline__ uint32_t inst() const { return key & 0xffffffu; }
    __device__ __forceinline__ uint32_t axis() const { return (key >> 24) & 3u; }
    __device__ __forceinline__ bool pos_dir() const { return ((key >> 26) & 1u) != 0; }
    __device__ __forceinline__ int32_t id(const FrameParams<float>& p) const { return p.inst[inst()].id; }
    __device__ __forceinline__ void set(uint32_t inst, int32_t, uint32_t axis, bool pos_dir) {
        key = (key & kFlagMask) | 0x80000000u | (pos_dir ? 1u << 26 : 0u) | (axis << 24) | inst;
    }
    // Compact hit-buffer kernels: per-pixel facts the store needs, kept in spare key
    // bits across the traversal instead of in registers of their own (set() keeps them)
    static constexpr uint32_t kMultiCand = 1u << 27; // more than one candidate: a hit is kMulti
    static constexpr uint32_t kNoSphere = 1u << 28;  // no sphere hit: a trivially reusable miss
    static constexpr uint32_t kReuse = 1u << 29;     // the record is reused (instance field: the object)
    static constexpr uint32_t kFlagMask = kMultiCand | kNoSphere | kReuse;
};

// World normal of the nearest hit: R n_local with n_local = sign e_axis
// opposing the unmirrored local direction (traversal.cpp:214-222, renderer.cpp:89).
template <typename Real> __device__ __forceinline__ void best_normal(const FrameParams<Real>& p, const Best<Real>& b, Real n[3]) {
    const DevInstance<Real>& in = p.inst[b.inst()];
    const uint32_t axis = b.axis();
    if constexpr (sizeof(Real) == 8) {
        // the reference's Mat3 * Vec3 (math.hpp:121-125), operand order kept
        Real nl[3] = {Real(0), Real(0), Real(0)};
        nl[axis] = b.pos_dir() ? Real(-1) : Real(1);
        for (int k = 0; k < 3; ++k) n[k] = in.R[3 * k] * nl[0] + in.R[3 * k + 1] * nl[1] + in.R[3 * k + 2] * nl[2];
    } else {
        // FP32: +-column `axis` of R, selected (the products with the one-hot local
        // normal are exact; the compact hit buffer expands records the same way)
        for (int k = 0; k < 3; ++k) n[k] = b.pos_dir() ? -in.R[3 * k + axis] : in.R[3 * k + axis];
    }
}

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
        s.hit = (d2 < in.r2 * 1.00001f + 1e-12f) && (s.tc + in.r * 1.00001f >= 0.0f);
        const float tb = s.tc - sqrtf(fmaxf(in.r2 - d2, 0.0f)) - 1e-5f * (fabsf(s.tc) + in.r);
        s.tb = fmaxf(tb, 0.0f);
    }
    return s;
}

// FP32 sphere test from the cull table (same conservative form as above).
__device__ __forceinline__ SphereRes<float> sphere_test(const float4 c, const float d[3]) {
    SphereRes<float> s;
    s.tc = c.x * d[0] + c.y * d[1] + c.z * d[2];
    const float px = c.x - s.tc * d[0], py = c.y - s.tc * d[1], pz = c.z - s.tc * d[2];
    const float d2 = px * px + py * py + pz * pz;
    const float r2 = c.w * c.w;
    s.hit = (d2 < r2 * 1.00001f + 1e-12f) && (s.tc + c.w * 1.00001f >= 0.0f);
    const float tb = s.tc - sqrtf(fmaxf(r2 - d2, 0.0f)) - 1e-5f * (fabsf(s.tc) + c.w);
    s.tb = fmaxf(tb, 0.0f);
    return s;
}

// Sphere test of instance i: FP64 from the instance record (reference order),
// FP32 from the cull table.
template <typename Real>
__device__ __forceinline__ SphereRes<Real> sphere_of(const FrameParams<Real>& p, uint32_t i, const Real d[3]) {
    if constexpr (sizeof(Real) == 8)
        return sphere_test(p.inst[i], d);
    else
        return sphere_test(__ldg(p.cull + i), d);
}

// FP64 camera-space direction of pixel (px, py), unnormalised (z = -1): the
// reference's NDC (renderer.cpp:19-21) is ((px + 0.5) / W) * 2 - 1 =
// (2 px + 1 - W) / W. The numerator is an exact integer, so a component is
// exactly zero iff the reference's is (its quotient is never within an ulp of
// 0.5 otherwise: the distance is >= 1/2W), and zero-direction rays stay zero;
// elsewhere the value is within a few FP64 ulp of the reference's, far below the
// FP32 rounding. The FP32 kernel forms each instance's local direction from it
// in FP64 and rounds once (a plane entry t = (A + i s) / d_a is only as accurate
// as the small component d_a), without normalising: a pixel's traversals all run
// in the same units (t_world = t |u|), recomputed per candidate from (px, py)
// instead of being held in registers across the candidate loop.
template <typename Real>
__device__ __forceinline__ void camera_dir_f64(const FrameParams<Real>& p, int px, int py, double& dcx, double& dcy) {
    dcx = static_cast<double>(2 * px + 1 - p.width) * p.d_kx;
    dcy = static_cast<double>(p.height - 2 * py - 1) * p.d_ky;
}

// ---- FP32 tile culling --------------------------------------------------------
// All rays of an 8x4 tile leave the camera inside one cone (axis: the tile's
// centre direction; half-angle: the widest corner). A bounding sphere that
// misses the (margin-inflated) cone misses every ray of the tile, so each warp
// tests the instances once per tile (lane i takes instances i, i+32, ...) and
// the per-ray sphere pass only visits the ballot-compacted survivors.
struct TileCone {
    float a[3];       // world axis (unit)
    float cos_a, sin_a;
};

// Cone of the pixel-centre rays of the w x h pixel region at (x0, y0).
template <typename Real>
__device__ __forceinline__ TileCone region_cone(const FrameParams<Real>& p, int x0, int y0, float w, float h) {
    const float inv_w2 = static_cast<float>(p.inv_w2), inv_h2 = static_cast<float>(p.inv_h2);
    const float sx = static_cast<float>(p.sx), sy = static_cast<float>(p.sy);
    const float cxs = fmaf(static_cast<float>(x0) + 0.5f * w, inv_w2, -1.0f) * sx;
    const float cys = fmaf(-(static_cast<float>(y0) + 0.5f * h), inv_h2, 1.0f) * sy;
    const float cn = rsqrtf(cxs * cxs + cys * cys + 1.0f);
    const float ax = cxs * cn, ay = cys * cn, az = -cn;
    // the four corner rays, one per lane (lane & 3; the whole warp calls this),
    // combined by a two-step butterfly max
    float smax;
    {
        const uint32_t k = threadIdx.x & 3u;
        const float xs = fmaf(static_cast<float>(x0) + ((k & 1u) ? w - 0.5f : 0.5f), inv_w2, -1.0f) * sx;
        const float ys = fmaf(-(static_cast<float>(y0) + ((k & 2u) ? h - 0.5f : 0.5f)), inv_h2, 1.0f) * sy;
        const float n = rsqrtf(xs * xs + ys * ys + 1.0f);
        const float bx = xs * n, by = ys * n, bz = -n;
        // |a x b| = sin of the angle (accurate for small angles, unlike 1 - cos)
        const float cx = ay * bz - az * by, cy = az * bx - ax * bz, cz = ax * by - ay * bx;
        smax = sqrtf(cx * cx + cy * cy + cz * cz);
        smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, 1));
        smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, 2));
    }
    TileCone c;
    c.sin_a = fminf(1.0f, smax * 1.01f + 1e-6f);
    c.cos_a = sqrtf(fmaxf(0.0f, 1.0f - c.sin_a * c.sin_a));
    for (int k = 0; k < 3; ++k)
        c.a[k] = static_cast<float>(p.C[3 * k]) * ax + static_cast<float>(p.C[3 * k + 1]) * ay +
                 static_cast<float>(p.C[3 * k + 2]) * az;
    return c;
}

// The same cone computed by one thread (the culling pre-pass's per-tile masks):
// the four corner rays in a loop instead of across lanes, the same arithmetic.
template <typename Real>
__device__ __forceinline__ TileCone region_cone_serial(const FrameParams<Real>& p, int x0, int y0, float w, float h) {
    const float inv_w2 = static_cast<float>(p.inv_w2), inv_h2 = static_cast<float>(p.inv_h2);
    const float sx = static_cast<float>(p.sx), sy = static_cast<float>(p.sy);
    const float cxs = fmaf(static_cast<float>(x0) + 0.5f * w, inv_w2, -1.0f) * sx;
    const float cys = fmaf(-(static_cast<float>(y0) + 0.5f * h), inv_h2, 1.0f) * sy;
    const float cn = rsqrtf(cxs * cxs + cys * cys + 1.0f);
    const float ax = cxs * cn, ay = cys * cn, az = -cn;
    float smax = 0.0f;
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k) {
        const float xs = fmaf(static_cast<float>(x0) + ((k & 1u) ? w - 0.5f : 0.5f), inv_w2, -1.0f) * sx;
        const float ys = fmaf(-(static_cast<float>(y0) + ((k & 2u) ? h - 0.5f : 0.5f)), inv_h2, 1.0f) * sy;
        const float n = rsqrtf(xs * xs + ys * ys + 1.0f);
        const float bx = xs * n, by = ys * n, bz = -n;
        const float cx = ay * bz - az * by, cy = az * bx - ax * bz, cz = ax * by - ay * bx;
        smax = fmaxf(smax, sqrtf(cx * cx + cy * cy + cz * cz));
    }
    TileCone c;
    c.sin_a = fminf(1.0f, smax * 1.01f + 1e-6f);
    c.cos_a = sqrtf(fmaxf(0.0f, 1.0f - c.sin_a * c.sin_a));
    for (int k = 0; k < 3; ++k)
        c.a[k] = static_cast<float>(p.C[3 * k]) * ax + static_cast<float>(p.C[3 * k + 1]) * ay +
                 static_cast<float>(p.C[3 * k + 2]) * az;
    return c;
}

template <typename Real> __device__ __forceinline__ TileCone tile_cone(const FrameParams<Real>& p, int x0, int y0) {
    return region_cone(p, x0, y0, static_cast<float>(kTileW), static_cast<float>(kTileH));
}

__device__ __forceinline__ bool cone_candidate(const float4 in, const TileCone& c) {
    const float lx = in.x, ly = in.y, lz = in.z;
    const float dist2 = lx * lx + ly * ly + lz * lz;
    const float r = in.w * 1.001f + 1e-5f * sqrtf(dist2) + 1e-6f;
    if (dist2 <= r * r) return true; // camera inside the (inflated) sphere
    // Conservative for the reference's sphere test (renderer.cpp:25-43), which
    // counts a hit when the ray's infinite line passes within r of the centre
    // and t_c + r >= 0 -- also for a chord wholly behind the camera. So: the
    // lateral distance is taken to the double cone (|s|), and a sphere behind
    // the apex is dropped only if even the most favourable direction of the
    // cone has t_c = L.d < -r.
    const float s = lx * c.a[0] + ly * c.a[1] + lz * c.a[2];
    const float qx = ly * c.a[2] - lz * c.a[1], qy = lz * c.a[0] - lx * c.a[2], qz = lx * c.a[1] - ly * c.a[0];
    const float perp = sqrtf(qx * qx + qy * qy + qz * qz);
    if (perp * c.cos_a - fabsf(s) * c.sin_a > r) return false; // outside the lateral surface
    return s * c.cos_a + perp * c.sin_a >= -r;                 // max over the cone of L.d, against -r
}

template <typename Real, bool kAov, bool kCompact>
__device__ __forceinline__ void trace_candidate(const FrameParams<Real>& p, uint32_t i, const Real dw[3], int px,
                                                int py, Best<Real>& best, uint32_t& traversals, uint32_t& fetches,
                                                BlockStack& stack) {
    const DevInstance<Real>& in = p.inst[i];
    if (!in.valid_model) return;
    ++traversals;
    Real ld[3];
    Real t;
    uint32_t axis, attr, parent, level, vox[3];
    if constexpr (sizeof(Real) == 8) {
        // d' = R^T d  (math.hpp:221-224, Mat3*Vec3 row order)
        LocalRay<Real> lr;
        for (int k = 0; k < 3; ++k) lr.d[k] = in.M[3 * k] * dw[0] + in.M[3 * k + 1] * dw[1] + in.M[3 * k + 2] * dw[2];
        setup_root(lr, in.A_lo, in.A_hi, in.zflags, in.zbits);
        TravHit<Real> h;
        NoLog nolog;
        const bool hit = (VXA_F64_SPLIT && lr.zero == 0) ? traverse_model<Real, NoLog, false>(in.model, lr, h, nolog)
                                                         : traverse_model(in.model, lr, h, nolog);
        fetches += h.fetches;
        if (!hit) return;
        for (int k = 0; k < 3; ++k) ld[k] = lr.d[k];
        t = h.t, axis = h.axis, attr = h.attr, parent = h.parent, level = h.level;
        if constexpr (kAov) path_to_voxel(h.path, h.level, vox);
    } else {
        float d[3];
        double dd[3];
        {
            double dcx, dcy;
            camera_dir_f64(p, px, py, dcx, dcy);
            for (int k = 0; k < 3; ++k) {
                dd[k] = fma(in.Md[3 * k], dcx, in.Md[3 * k + 1] * dcy) - in.Md[3 * k + 2];
                d[k] = static_cast<float>(dd[k]);
            }
        }
        // Content sphere (conservative, margin included): every leaf lies inside
        // it, so a ray whose line misses it -- or that is outside it and moving
        // away -- hits nothing here; the traversal is skipped. FP64 unit-cube
        // coordinates: origin -U_lo (plus residual) relative to the centre 0.5.
        if (in.model.content_r2 < 0.75f) {
            double qq = 0.0, qw = 0.0, ww = 0.0;
            for (int k = 0; k < 3; ++k) {
                const double q = -(static_cast<double>(in.U_lo[k]) + static_cast<double>(in.Ur_lo[k])) - 0.5;
                const double w = dd[k] * in.ih2[k];
                qq = fma(q, q, qq);
                qw = fma(q, w, qw);
                ww = fma(w, w, ww);
            }
            // squared line distance qq - qw^2/ww > r2, without the division (ww > 0;
            // homogeneous in w, so the unnormalised direction serves)
            const double r2 = static_cast<double>(in.model.content_r2);
            if (fma(qq, ww, -qw * qw) > r2 * ww || (qw > 0.0 && qq > r2)) return;
        }
        FastRay fr;
        // Only a hit at t <= best.t can change the nearest (t, id) (ties go to
        // the lower id), so subtrees entered beyond best.t are pruned.
        const float t_lim = best.have() ? nextafterf(static_cast<float>(best.t), __int_as_float(0x7f800000))
                                        : __int_as_float(0x7f800000);
        if (!fast_setup(fr, d, in.U_lo, in.U_hi, in.Ur_lo, in.Ur_hi, in.h2, in.zflags, in.zbits, t_lim)) return;
        FastHit h;
        bool hit;
        if constexpr (kCompact) {
            CompactNodes nodes{in.model.cwords};
            if constexpr (VXA_SMEM_TOP > 0) {
                if (in.model.cwords == p.top_words) {
                    nodes.top_base = stack.base_top;
                    nodes.top_n = p.top_n;
                }
            }
#if VXA_ZERO_SPLIT
            // rays with a zero local direction component are rare: they take the
            // general copy, every other ray a loop without the zero conventions
            if (fr.zero)
                hit = traverse_fast<kAov, true>(nodes, static_cast<int>(in.model.depth), fr, h, stack);
            else if constexpr (VXA_POSLOOP)
                hit = traverse_pos<kAov>(nodes, static_cast<int>(in.model.depth), fr, h, stack);
            else
                hit = traverse_fast<kAov, false>(nodes, static_cast<int>(in.model.depth), fr, h, stack);
#else
            if (VXA_POSLOOP && !fr.zero)
                hit = traverse_pos<kAov>(nodes, static_cast<int>(in.model.depth), fr, h, stack);
            else
                hit = traverse_fast<kAov>(nodes, static_cast<int>(in.model.depth), fr, h, stack);
#endif
        }
        else if (VXA_POSLOOP && !fr.zero)
            hit = traverse_pos<kAov>(WideNodes{in.model.words, in.model.side}, static_cast<int>(in.model.depth), fr, h,
                                     stack);
        else
            hit = traverse_fast<kAov>(WideNodes{in.model.words, in.model.side}, static_cast<int>(in.model.depth), fr, h,
                                      stack);
        fetches += h.fetches;
        if (!hit) return;
        for (int k = 0; k < 3; ++k) ld[k] = d[k], vox[k] = h.vox[k];
        t = h.t, axis = h.axis, attr = h.attr, parent = h.parent, level = h.level;
    }
    if (!best.have() || t < best.t || (t == best.t && in.id < best.id(p))) {
        best.set(i, in.id, axis, ld[axis] > Real(0));
        best.t = t;
        best.attr = attr;
        if constexpr (kAov) {
            best.parent = parent;
            best.level = level;
            best.vox[0] = vox[0], best.vox[1] = vox[1], best.vox[2] = vox[2];
        }
    }
}

// Direct readback of one finished super-tile (called by the whole warp that
// finished its last tile): its RGB8 rows, written to the device image by the
// tiles' warps, are copied into the caller's page-locked host image (mapped)
// with 16-byte stores over PCIe -- 192-byte row segments, 64-byte aligned --
// while the rest of the frame renders. Loads bypass L1 (other SMs wrote the
// rows). Out of line, with scalar arguments: the frame kernel's register
// allocation is not disturbed by this cold path.
static __device__ __noinline__ void flush_rows(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint32_t row_bytes,
                                        uint32_t seg_bytes, uint32_t rows, uint32_t lane) {
    __threadfence(); // every lane reads after lane 0's acquire
    if ((seg_bytes & 15u) == 0 && (row_bytes & 15u) == 0 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0 &&
        (reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
        const uint32_t per_row = seg_bytes >> 4, n = per_row * rows;
        constexpr uint32_t kBatch = 4; // loads in flight per lane before their stores
        for (uint32_t base = 0; base < n; base += 32u * kBatch) {
            uint4 v[kBatch];
#pragma unroll
            for (uint32_t j = 0; j < kBatch; ++j) {
                const uint32_t i = base + lane + 32u * j, r = i / per_row;
                if (i < n) v[j] = __ldcg(reinterpret_cast<const uint4*>(src + r * row_bytes + 16u * (i - r * per_row)));
            }
#pragma unroll
            for (uint32_t j = 0; j < kBatch; ++j) {
                const uint32_t i = base + lane + 32u * j, r = i / per_row;
                if (i < n) *reinterpret_cast<uint4*>(dst + r * row_bytes + 16u * (i - r * per_row)) = v[j];
            }
        }
    } else {
        for (uint32_t r = 0; r < rows; ++r)
            for (uint32_t b = lane; b < seg_bytes; b += 32u) dst[r * row_bytes + b] = __ldcg(src + r * row_bytes + b);
    }
}

template <typename Real>
__device__ __forceinline__ void flush_super_rgb(const FrameParams<Real>& p, uint32_t s, uint32_t lane) {
    const uint32_t sy = super_row(p, s), sx = s - sy * p.n_super_x;
    const uint32_t x0 = sx * kSuper, y0 = sy * kSuper;
    const uint32_t w = min(static_cast<uint32_t>(kSuper), static_cast<uint32_t>(p.width) - x0);
    const uint32_t h = min(static_cast<uint32_t>(kSuper), static_cast<uint32_t>(p.height) - y0);
    const size_t o0 = 3 * (static_cast<size_t>(y0) * static_cast<size_t>(p.width) + x0);
    flush_rows(p.rgb + o0, p.rgb_host + o0, 3u * static_cast<uint32_t>(p.width), 3u * w, h, lane);
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

// kHbo: 0 no hit buffer, 1 48-byte host-layout records, 2 16-byte records (FP32)
// kDirect: direct synchronous readback (p.super_done / p.rgb_host set; no AOV or
// hit buffer) -- its own instantiation, so the other kernels carry none of it
template <typename Real, bool kAov, int kHbo, bool kCompact, bool kDirect = false>
__global__ void __launch_bounds__(kBlock, sizeof(Real) == 4 ? VXA_MIN_BLOCKS : VXA_MIN_BLOCKS_F64) frame_kernel(const __grid_constant__ FrameParams<Real> p) {
    extern __shared__ uint2 smem_stack[]; // FP32 traversal stack: [level][thread]
    __shared__ uint16_t s_list[kWarps][kListCap];
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    // rays and sphere tests per frame are known on the host (pixels x objects)
    uint32_t n_trav = 0, n_reuse = 0, n_fetch = 0, n_leaf = 0;
    const uint32_t n = p.n_inst;
    BlockStack stack;
    stack.base = static_cast<uint32_t>(__cvta_generic_to_shared(smem_stack)) + kStackEntry * threadIdx.x;
#if VXA_STACK_TEN && VXA_STACK_LAYOUT == 2
    stack.base_ten = static_cast<uint32_t>(__cvta_generic_to_shared(smem_stack)) + 8u * kBlock * stack_levels(p.max_depth) +
                     4u * threadIdx.x;
    asm volatile("" : "+r"(stack.base_ten));
#endif
    stack.base_top = 0;
    if constexpr (sizeof(Real) == 4 && VXA_SMEM_TOP > 0) {
        // Stage the scene model's first VXA_SMEM_TOP node words (its top levels, BFS
        // order) into shared memory behind the stack: one bulk copy (TMA engine)
        // completing on an mbarrier, issued by one thread.
        __shared__ __align__(8) unsigned long long top_bar;
        const uint32_t top = static_cast<uint32_t>(__cvta_generic_to_shared(
            reinterpret_cast<unsigned char*>(smem_stack) + kStackBytes * kBlock * stack_levels(p.max_depth)));
        stack.base_top = top;
        if (p.top_words != nullptr && p.top_n > 0) {
            const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&top_bar));
            const uint32_t bytes = 4u * p.top_n;
            if (threadIdx.x == 0) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(top),
                    "l"(p.top_words), "r"(bytes), "r"(bar)
                    : "memory");
            }
            __syncthreads(); // the barrier is initialised before anyone waits on it
            uint32_t done = 0;
            while (!done) {
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done)
                    : "r"(bar)
                    : "memory");
            }
        }
    }
    // opaque to the optimiser: kept in a register instead of being re-derived
    // from %tid / the CTA window (6 instructions) on every push
    asm volatile("" : "+r"(stack.base));
#if VXA_PDL
    // launched as a programmatic dependent of the culling pre-pass: everything
    // above overlapped its tail; the lists, the order and the tile counter are
    // read only after it completed (a no-op for an ordinary launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    const uint16_t* const list = s_list[warp];

    // band (banded readback) or super-tile (direct readback) of the warp's previous tile
    int prev_band = -1;
    while (true) {
        __syncwarp();
        if (prev_band >= 0) {
            // the previous tile's RGB8 bytes are visible before its count moves: the
            // warp barrier orders the lanes' stores before lane 0's gpu-scope release
            // increment (cumulative) -- one release per tile, not 32 fences.
            if constexpr (kDirect) {
                // direct readback: the warp that completes a super-tile (its count's
                // acquire sees every other tile's release) stores its rows to the host
                uint32_t last = 0;
                if (lane == 0) {
                    uint32_t old;
                    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                                 : "=r"(old)
                                 : "l"(p.super_done + prev_band)
                                 : "memory");
                    last = old == static_cast<uint32_t>(kTilesPerSuper) - 1u ? 1u : 0u;
                }
                if (__shfl_sync(0xffffffffu, last, 0)) flush_super_rgb(p, static_cast<uint32_t>(prev_band), lane);
            } else if (lane == 0) {
                // banded readback: the copy engine starts a band's D2H when its count is
                // complete. (Adding a warp's tiles per band once it leaves the band costs
                // fewer releases but signals the bands late: the D2H overlapped less,
                // DESIGN.md §11.)
                unsigned int* const cnt = p.band_done + prev_band;
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
            }
        }
        uint32_t tile = 0;
        if (lane == 0) tile = atomicAdd(p.tile_counter, 1u);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= p.n_tiles) break;
        const uint32_t st_k = tile / kTilesPerSuper, wt = tile % kTilesPerSuper;
        const uint32_t st = p.super_order != nullptr ? __ldg(p.super_order + st_k) : st_k;
        const uint32_t s = st * static_cast<uint32_t>(p.world) + static_cast<uint32_t>(p.rank);
        const uint32_t sy = super_row(p, s), sx = s - sy * p.n_super_x;
        if (p.band_done != nullptr) prev_band = static_cast<int>(sy / p.band_rows);
        if constexpr (kDirect) prev_band = static_cast<int>(s);
        const int tx0 = static_cast<int>(sx * kSuper + (wt % (kSuper / kTileW)) * kTileW);
        const int ty0 = static_cast<int>(sy * kSuper + (wt / (kSuper / kTileW)) * kTileH);
        int px = tx0 + static_cast<int>(lane % kTileW);
        int py = ty0 + static_cast<int>(lane / kTileW);

        // ---- tile candidate list (culling on). Conservative: a sphere missing the
        // inflated tile cone misses every ray of the tile, in either kernel; the
        // list keeps instance order, so the FP64 kernel's candidates, their order
        // and its ties are those of the per-ray pass over every instance.
        uint32_t list_n = 0xffffffffu; // 0xffffffff: per-ray pass over every instance
        {
            if (p.culling && n <= 0xffffu) {
                // source: the super-tile's candidate list when the pre-pass ran
                const uint16_t* src = nullptr;
                uint32_t src_n = n;
                if (p.super_list != nullptr) {
                    const uint32_t c = __ldg(p.super_count + st);
                    if (c != 0xffffffffu) src = p.super_list + static_cast<size_t>(st) * p.super_cap, src_n = c;
                }
                // the pre-pass's per-tile mask over the super-tile's list when it has one
                // (the same cone tests, done once per tile by one thread instead of per warp)
                const bool masked = src != nullptr && p.tile_mask != nullptr && src_n <= kListCap;
                const unsigned long long tmask =
                    masked ? __ldg(p.tile_mask + static_cast<size_t>(st) * kTilesPerSuper + wt) : 0ull;
                TileCone cone{};
                if (!masked) cone = tile_cone(p, tx0, ty0); // warp-uniform branch (the cone shuffles)
                uint32_t cnt = 0;
                for (uint32_t base = 0; base < src_n; base += 32) {
                    const uint32_t j = base + lane;
                    const uint32_t i = j < src_n ? (src ? __ldg(src + j) : j) : 0u;
                    const bool c = j < src_n && (masked ? ((tmask >> j) & 1ull) != 0 : cone_candidate(__ldg(p.cull + i), cone));
                    const uint32_t m = __ballot_sync(0xffffffffu, c);
                    const uint32_t pos = cnt + __popc(m & ((1u << lane) - 1u));
                    if (c && pos < kListCap) s_list[warp][pos] = static_cast<uint16_t>(i);
                    cnt += __popc(m);
                }
                __syncwarp();
                if (cnt <= kListCap) list_n = cnt;
            }
        }
        // warp-uniform: no lane of the tile leaves the frame (the RGB8 store gathers across lanes)
        const bool tile_inside = tx0 + kTileW <= p.width && ty0 + kTileH <= p.height;
        if (px >= p.width || py >= p.height) continue;
        // the tile origin packed in one register; the pixel's coordinates and
        // index are rebuilt from it where needed instead of staying live
        uint32_t txy = (static_cast<uint32_t>(ty0) << 16) | static_cast<uint32_t>(tx0);
        const auto pixel_xy = [&](int& x, int& y) {
            asm volatile("" : "+r"(txy));
            x = static_cast<int>(txy & 0xffffu) + static_cast<int>(lane % kTileW);
            y = static_cast<int>(txy >> 16) + static_cast<int>(lane / kTileW);
        };
        const auto pixel_index = [&]() {
            int x, y;
            pixel_xy(x, y);
            return static_cast<size_t>(y) * static_cast<size_t>(p.width) + static_cast<size_t>(x);
        };

        // ---- primary ray (renderer.cpp:11-23)
        Real dw[3];
        float ulen = 1.0f; // FP32: |u| -- the pixel's traversal units to world units (t_world = t |u|)
        if constexpr (sizeof(Real) == 8) {
            const double ndc_x = (px + 0.5) / p.width * 2.0 - 1.0;
            const double ndc_y = 1.0 - (py + 0.5) / p.height * 2.0;
            const double dc[3] = {ndc_x * p.tan_half * p.aspect, ndc_y * p.tan_half, -1.0};
            Real w[3];
            for (int k = 0; k < 3; ++k) w[k] = p.C[3 * k] * dc[0] + p.C[3 * k + 1] * dc[1] + p.C[3 * k + 2] * dc[2];
            const double len = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
            for (int k = 0; k < 3; ++k) dw[k] = w[k] / len;
        } else {
            const float dcx = fmaf(static_cast<float>(px) + 0.5f, p.inv_w2, -1.0f) * p.sx;
            const float dcy = fmaf(-(static_cast<float>(py) + 0.5f), p.inv_h2, 1.0f) * p.sy;
            const float uu = fmaf(dcx, dcx, fmaf(dcy, dcy, 1.0f));
            const float rn = rsqrtf(uu);
            ulen = uu * rn;
            for (int k = 0; k < 3; ++k) dw[k] = (p.C[3 * k] * dcx + p.C[3 * k + 1] * dcy - p.C[3 * k + 2]) * rn;
        }
        // world-units t of the best hit: the FP32 kernel traverses along the
        // unnormalised direction u, whose parameter is t_world / |u|
        const auto world_t = [&](Real t) { return sizeof(Real) == 8 ? t : static_cast<Real>(static_cast<float>(t) * ulen); };

        // ---- sphere pass: count hits, remember the single hit (HBO rule)
        uint32_t n_hits = 0, only = 0;
        unsigned long long hitmask = 0; // list mode: bit k = s_list[warp][k] hit
        // list mode: 1 + the (t_center, index) minimum of the hits -- the first candidate
        // of the sorted order, so its pick needs no second pass over the hits
        uint32_t first_pick = 0;
        if (list_n != 0xffffffffu) {
            Real first_tc = Real(0);
            for (uint32_t k = 0; k < list_n; ++k) {
                const SphereRes<Real> sr = sphere_of(p, list[k], dw);
                if (sr.hit) {
                    hitmask |= 1ull << k;
                    if (first_pick == 0 || sr.tc < first_tc) first_pick = k + 1, first_tc = sr.tc;
                }
            }
            n_hits = __popcll(hitmask);
            if (n_hits) only = list[__ffsll(hitmask) - 1];
        } else if (p.sphere_pass) {
            for (uint32_t i = 0; i < n; ++i) {
                if (sphere_of(p, i, dw).hit) {
                    if (n_hits == 0) only = i;
                    ++n_hits;
                }
            }
        }

        Best<Real> best;
        // per-pixel traversal / fetch counts (AOV kernels); otherwise the traversals
        // count straight into the warp's totals (two fewer live registers)
        uint32_t px_trav = 0, px_fetch = 0, kind = kMiss;
        uint32_t& traversals = kAov ? px_trav : n_trav;
        uint32_t& fetches = kAov ? px_fetch : n_fetch;
        bool reused = false;
        bool single_trace = false;
        constexpr bool compact_hbo = sizeof(Real) == 4 && kHbo == 2;
        if constexpr (kHbo) {
            if (!p.camera_dirty && n_hits == 1) {
                const DevInstance<Real>& o = p.inst[only];
                // a dirty object is never reused: its record is not even read
                bool same = false;
                if (!o.dirty) {
                    if (compact_hbo) {
                        // only kind and id decide; a reused record is read again for shading
                        // (nothing of it stays live across the traversal)
                        const HitRec16 prev16 = reinterpret_cast<const HitRec16*>(p.hbo)[pixel_index()];
                        same = (prev16.meta & 3u) == kSingle && prev16.object_id == o.id;
                    } else {
                        const HitRec* const pr = reinterpret_cast<const HitRec*>(p.hbo) + pixel_index();
                        same = pr->kind == kSingle && pr->object_id == o.id;
                    }
                }
                if (same) {
                    reused = true;
                } else {
                    single_trace = true; // "trace just this SVO"
                }
            }
        }
        if constexpr (compact_hbo && !kAov) {
            // what the store needs from the sphere pass, in spare bits of the best key
            if (reused) best.key = Best<Real>::kReuse | only; // n_hits == 1: the object
            if (n_hits == 0) best.key |= Best<Real>::kNoSphere;
        }

        if (!reused) {
            // One traversal call site; the candidate order comes from a small
            // state machine (keeps a single inlined copy of the traversal).
            enum { kOne, kListSorted, kListIdOrder, kAllSorted, kAllIdOrder } mode;
            uint32_t n_cand;
            if (single_trace) {
                mode = kOne, n_cand = 1;
            } else if (list_n != 0xffffffffu) {
                mode = p.sorting ? kListSorted : kListIdOrder, n_cand = n_hits;
            } else if (p.sorting) {
                mode = kAllSorted, n_cand = p.culling ? n_hits : n;
            } else {
                mode = kAllIdOrder, n_cand = p.culling ? n_hits : n;
            }
            if constexpr (compact_hbo && !kAov)
                if (n_cand > 1) best.key |= Best<Real>::kMultiCand;
            unsigned long long rem = hitmask; // list modes: hit bits not yet visited
            Real last_tc = -pos_inf<Real>();  // kAllSorted: last (t_center, index) taken
            int last_i = -1;
            uint32_t next_i = mode == kListSorted ? first_pick : 0u; // kAllIdOrder cursor; kListSorted: the pending first pick
            bool one_left = true;
            while (true) {
                uint32_t cand = 0;
                Real cand_tb = Real(0);
                bool found = false;
                if (mode == kOne) {
                    found = one_left, cand = only, one_left = false;
                } else if (mode == kListSorted) {
                    // (t_center, index) minimum over the remaining hit bits. The first
                    // one is the sphere pass's (its t_boundary only matters once there
                    // is a best hit: none yet).
                    int kb = -1;
                    Real tcb = Real(0);
                    if (next_i != 0) {
                        kb = static_cast<int>(next_i) - 1;
                        next_i = 0;
                    } else {
                        // A candidate whose t_boundary is beyond the best hit is skipped
                        // whenever its turn comes (the best t only decreases), so it
                        // leaves the set now: the passes stop once nothing left can be
                        // traced, instead of visiting every skipped candidate in order.
                        const Real bt = best.have() ? world_t(best.t) : pos_inf<Real>();
                        for (unsigned long long it = rem; it; it &= it - 1) {
                            const int k = __ffsll(it) - 1;
                            const SphereRes<Real> sr = sphere_of(p, list[k], dw);
                            if (bt < sr.tb) {
                                rem &= ~(1ull << k);
                                continue;
                            }
                            if (kb < 0 || sr.tc < tcb) kb = k, tcb = sr.tc, cand_tb = sr.tb;
                        }
                    }
                    if (kb >= 0) found = true, cand = list[kb], rem &= ~(1ull << kb);
                } else if (mode == kListIdOrder) {
                    if (rem) found = true, cand = list[__ffsll(rem) - 1], rem &= rem - 1;
                } else if (mode == kAllSorted) {
                    int k = -1;
                    Real k_tc = Real(0);
                    const Real bt = best.have() ? world_t(best.t) : pos_inf<Real>();
                    for (uint32_t i = 0; i < n; ++i) {
                        const SphereRes<Real> sr = sphere_of(p, i, dw);
                        if (p.culling && !sr.hit) continue;
                        const bool after = sr.tc > last_tc || (sr.tc == last_tc && static_cast<int>(i) > last_i);
                        if (!after) continue;
                        // skipped whenever it comes up (sphere hits: t_boundary; the
                        // no-culling order's misses carry 0 and are never skipped)
                        if (sr.hit && bt < sr.tb) continue;
                        if (k < 0 || sr.tc < k_tc) k = static_cast<int>(i), k_tc = sr.tc, cand_tb = sr.hit ? sr.tb : Real(0);
                    }
                    if (k >= 0) found = true, cand = static_cast<uint32_t>(k), last_tc = k_tc, last_i = k;
                } else {
                    while (next_i < n && p.culling && !sphere_of(p, next_i, dw).hit) ++next_i;
                    if (next_i < n) found = true, cand = next_i++;
                }
                if (!found) break;
                // sorted orders: skip (do not break) when the best hit is nearer than the
                // candidate's sphere (renderer.cpp:70-72); id orders carry t_boundary = 0
                if ((mode == kListSorted || mode == kAllSorted) && best.have() && world_t(best.t) < cand_tb) continue;
                pixel_xy(px, py);
                trace_candidate<Real, kAov, kCompact>(p, cand, dw, px, py, best, traversals, fetches, stack);
            }
            if constexpr (!(compact_hbo && !kAov)) {
                if (best.have()) kind = n_cand > 1 ? kMulti : kSingle;
                if constexpr (kHbo) {
                    if (!p.camera_dirty && p.culling && n_hits == 0) reused = true; // trivial reuse of a miss
                }
            }
        }
        if constexpr (kAov) {
            n_trav += px_trav;
            n_fetch += px_fetch;
        }
        // compact hit buffer (production): the reuse facts come back from the key
        bool reuse_rec; // the record is reused as it is (reused with one sphere hit)
        if constexpr (compact_hbo && !kAov) {
            const uint32_t f = best.key;
            reuse_rec = (f & Best<Real>::kReuse) != 0;
            kind = (f >> 31) ? ((f & Best<Real>::kMultiCand) ? kMulti : kSingle) : kMiss;
            reused = reuse_rec || (!p.camera_dirty && p.culling && (f & Best<Real>::kNoSphere) != 0);
        } else {
            reuse_rec = reused && n_hits == 1;
        }
        if (reused) ++n_reuse;

        // ---- shade + store
        uint32_t rgba;
        if constexpr (compact_hbo) {
            // 16-byte records: a reused record's normal is the object's current R
            // times its stored local normal (the object is not dirty)
            HitRec16 rec;
            if (reuse_rec) {
                rec = reinterpret_cast<const HitRec16*>(p.hbo)[pixel_index()];
            } else {
                rec.color = best.have() ? __ldg(p.inst[best.inst()].model.attrs + best.attr) : 0xff000000u;
                rec.t = best.have() ? static_cast<float>(world_t(best.t)) : 0.0f;
                rec.object_id = best.have() ? best.id(p) : -1;
                rec.meta = kind | (best.axis() << 2) | (best.pos_dir() ? 16u : 0u);
            }
            if ((rec.meta & 3u) == kMiss) {
                rgba = p.background;
            } else {
                Best<Real> b = best;
                if (reuse_rec) {
                    const uint32_t obj = (compact_hbo && !kAov) ? best.inst() : only;
                    b.set(obj, rec.object_id, (rec.meta >> 2) & 3u, (rec.meta & 16u) != 0);
                }
                Real nrm[3];
                best_normal(p, b, nrm);
                rgba = shade_rgba(rec.color, nrm, dw);
            }
            if (!reuse_rec) reinterpret_cast<HitRec16*>(p.hbo)[pixel_index()] = rec; // a reused record is unchanged
        } else if constexpr (kHbo == 1) {
            HitRec rec;
            if (reused && n_hits == 1) {
                rec = reinterpret_cast<const HitRec*>(p.hbo)[pixel_index()];
            } else {
                rec.color = best.have() ? __ldg(p.inst[best.inst()].model.attrs + best.attr) : 0xff000000u;
                rec.pad0 = 0;
                Real nrm[3] = {Real(0), Real(0), Real(0)};
                if (best.have()) best_normal(p, best, nrm);
                for (int k = 0; k < 3; ++k) rec.normal[k] = static_cast<double>(nrm[k]);
                rec.t = best.have() ? static_cast<double>(world_t(best.t)) : 0.0;
                rec.object_id = best.have() ? best.id(p) : -1;
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
            if (!(reused && n_hits == 1)) reinterpret_cast<HitRec*>(p.hbo)[pixel_index()] = rec; // a reused record is unchanged
        } else {
            if (best.have()) {
                const uint32_t color = __ldg(p.inst[best.inst()].model.attrs + best.attr);
                Real nrm[3];
                best_normal(p, best, nrm);
                rgba = shade_rgba(color, nrm, dw);
            } else {
                rgba = p.background;
            }
        }
        if (best.have()) ++n_leaf;
        const size_t pix = pixel_index();
        p.fb[pix] = rgba;
        if (p.rgb != nullptr) { // streamed frame: the readback's RGB8 bytes too (no pack pass)
            if (kTileW == 8 && tile_inside && (p.width & 3) == 0) {
                // A tile row is 8 pixels = 24 contiguous RGB8 bytes = six 4-byte words
                // (4-aligned: 3 (y W + x0) with W % 4 == 0 and x0 % 8 == 0). Lane j < 6
                // of each row gathers the two pixels its word covers (bytes 4j .. 4j+3
                // = pixels 4j/3 and 4j/3 + 1) and stores the word: 24 lanes x 4 B.
                const uint32_t r = lane >> 3, j = lane & 7u;
                const uint32_t q0 = (4u * j) / 3u;
                const uint32_t src0 = (r << 3) + min(q0, 7u), src1 = (r << 3) + min(q0 + 1u, 7u);
                const uint32_t v0 = __shfl_sync(0xffffffffu, rgba, src0);
                const uint32_t v1 = __shfl_sync(0xffffffffu, rgba, src1);
                const uint32_t j3 = j - 3u * (j / 3u);
                const uint32_t sel = j3 == 0 ? 0x4210u : (j3 == 1 ? 0x5421u : 0x6542u);
                if (j < 6u) {
                    const size_t row = static_cast<size_t>((txy >> 16) + r) * static_cast<size_t>(p.width) +
                                       static_cast<size_t>(txy & 0xffffu);
                    *reinterpret_cast<uint32_t*>(p.rgb + 3 * row + 4 * j) = __byte_perm(v0, v1, sel);
                }
            } else {
                uint8_t* o = p.rgb + 3 * pix;
                o[0] = static_cast<uint8_t>(rgba);
                o[1] = static_cast<uint8_t>(rgba >> 8);
                o[2] = static_cast<uint8_t>(rgba >> 16);
            }
        }

        if constexpr (kAov) {
            PixelAov a;
            a.t = best.have() ? static_cast<double>(world_t(best.t)) : 0.0;
            a.object_id = best.have() ? best.id(p) : (kHbo != 0 && reused && n_hits == 1 ? -2 : -1);
            a.node_index = best.parent;
            a.attr_index = best.attr;
            a.voxel[0] = best.vox[0];
            a.voxel[1] = best.vox[1];
            a.voxel[2] = best.vox[2];
            a.level = static_cast<uint8_t>(best.level);
            a.kind = static_cast<uint8_t>(kind);
            a.entry_axis = static_cast<uint8_t>(best.axis());
            a.pad0 = 0;
            a.traversals = traversals;
            a.node_fetches = fetches;
            a.pad1 = 0;
            reinterpret_cast<PixelAov*>(p.aov)[pix] = a;
        }
    }

    // multi-GPU: this thread's peer stores are performed system-wide before the
    // rank's completion flag (vxa_frame_close) can be written
    if (p.fence_sys) __threadfence_system();
    // warp-aggregated counters: traversals, reuse, node fetches, leaf hits
    const uint32_t vals[4] = {n_trav, n_reuse, n_fetch, n_leaf};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t v = __reduce_add_sync(0xffffffffu, vals[k]);
        if (lane == 0 && v) atomicAdd(p.counters + 2 + k, static_cast<unsigned long long>(v));
    }
}

// Longest-first order of the rank's super-tiles for the frame kernel's work
// queue: a counting sort by descending candidate count (overflowed lists first,
// empty ones last), run by the pre-pass's last block. Only the schedule
// changes -- every pixel's arithmetic is the same -- so the grid's tail is made
// of cheap tiles instead of whatever the screen order puts last. `count` was
// written by other blocks of the same grid: read through L2 (__ldcg), not the
// read-only path.
// With band_rows (a banded synchronous readback): super-tile rows in bands of
// band_rows, bands in screen order so they complete one after another, and
// longest-first inside each band so a band's slowest tiles start first. The
// bucket offsets come from a block-wide scan (up to 16 x 66 buckets).
__device__ __forceinline__ void order_by_count(const uint32_t* count, uint32_t n, uint32_t* order, uint32_t n_super_x,
                                               uint32_t band_rows) {
    constexpr uint32_t kPer = 66; // overflow, 64 .. 0 candidates
    constexpr uint32_t kBands = 16;
    constexpr uint32_t kMax = kPer * kBands;
    __shared__ uint32_t start[kMax];
    __shared__ uint32_t warp_sum[32];
    const uint32_t n_buckets = band_rows ? kMax : kPer;
    const auto bucket = [&](uint32_t i) {
        const uint32_t c = __ldcg(count + i);
        const uint32_t b = c == 0xffffffffu ? 0u : 65u - min(c, 64u);
        return band_rows ? min((i / n_super_x) / band_rows, kBands - 1) * kPer + b : b;
    };
    for (uint32_t b = threadIdx.x; b < n_buckets; b += blockDim.x) start[b] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&start[bucket(i)], 1u);
    __syncthreads();
    // exclusive scan: each thread a contiguous chunk, then the chunk totals across the block
    const uint32_t per = (n_buckets + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = min(threadIdx.x * per, n_buckets), b1 = min(b0 + per, n_buckets);
    uint32_t local = 0;
    for (uint32_t b = b0; b < b1; ++b) local += start[b];
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    uint32_t incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += v;
    }
    if (lane == 31) warp_sum[wid] = incl;
    __syncthreads();
    uint32_t base = 0;
    for (uint32_t w = 0; w < wid; ++w) base += warp_sum[w];
    uint32_t acc = base + incl - local;
    for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t c = start[b];
        start[b] = acc;
        acc += c;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) order[atomicAdd(&start[bucket(i)], 1u)] = i;
}

// Pre-pass for large scenes, one block per super-tile of this rank: its first
// warp cone-tests every instance against the super-tile's cone and writes the
// survivors (in instance order) to the super-tile's list; then (lists of <= 64
// entries) each thread tests one 8x4 tile's cone against that list and writes the
// tile's candidate mask, so the frame kernel's warps need no cone arithmetic.
// With p.super_order set, the grid's last block to finish (a ticket on `done`,
// which it resets) then writes the longest-first super-tile order.
template <typename Real>
__global__ void __launch_bounds__(128) super_cull_kernel(const __grid_constant__ FrameParams<Real> p,
                                                        uint16_t* __restrict__ list, uint32_t* __restrict__ count,
                                                        uint32_t* __restrict__ done) {
    // one block per super-tile: warp 0 builds its candidate list, then every thread
    // computes one 8x4 tile's mask over that list
    __shared__ uint16_t s_cand[kListCap];
    __shared__ uint32_t s_cnt;
    const uint32_t lane = threadIdx.x & 31u;
#if VXA_PDL
    asm volatile("griddepcontrol.launch_dependents;");
#endif
    if (blockIdx.x == 0 && threadIdx.x < 8) {
        // the frame kernel's work counter and (when asked) the frame's statistics start
        // at zero: the previous frame kernel is done (stream order), this frame's has
        // not started
        if (threadIdx.x == 0) *p.tile_counter = 0;
        if (p.reset_stats) p.counters[threadIdx.x] = 0;
    }
    const uint32_t st = blockIdx.x;
    const uint32_t s = st * static_cast<uint32_t>(p.world) + static_cast<uint32_t>(p.rank);
    const uint32_t sy = super_row(p, s);
    const int x0 = static_cast<int>((s - sy * p.n_super_x) * kSuper), y0 = static_cast<int>(sy * kSuper);
    if (threadIdx.x < 32) {
        const float w = static_cast<float>(min(kSuper, p.width - x0)), h = static_cast<float>(min(kSuper, p.height - y0));
        const TileCone cone = region_cone(p, x0, y0, w, h);
        uint16_t* out = list + static_cast<size_t>(st) * p.super_cap;
        uint32_t cnt = 0;
        for (uint32_t base = 0; base < p.n_inst; base += 32) {
            const uint32_t i = base + lane;
            const bool c = i < p.n_inst && cone_candidate(__ldg(p.cull + i), cone);
            const uint32_t m = __ballot_sync(0xffffffffu, c);
            const uint32_t pos = cnt + __popc(m & ((1u << lane) - 1u));
            if (c && pos < p.super_cap) out[pos] = static_cast<uint16_t>(i);
            if (c && pos < kListCap) s_cand[pos] = static_cast<uint16_t>(i);
            cnt += __popc(m);
        }
        if (lane == 0) {
            count[st] = cnt <= p.super_cap ? cnt : 0xffffffffu;
            s_cnt = cnt;
        }
    }
    __syncthreads();
    const uint32_t cnt = s_cnt;
    if (p.tile_mask != nullptr && cnt <= kListCap) {
        // tile wt of the super-tile: which entries of its list meet the tile's cone
        for (uint32_t wt = threadIdx.x; wt < kTilesPerSuper; wt += blockDim.x) {
            const int tx0 = x0 + static_cast<int>((wt % (kSuper / kTileW)) * kTileW);
            const int ty0 = y0 + static_cast<int>((wt / (kSuper / kTileW)) * kTileH);
            unsigned long long m = 0;
            if (tx0 < p.width && ty0 < p.height) {
                const TileCone tc =
                    region_cone_serial(p, tx0, ty0, static_cast<float>(kTileW), static_cast<float>(kTileH));
                for (uint32_t j = 0; j < cnt; ++j)
                    if (cone_candidate(__ldg(p.cull + s_cand[j]), tc)) m |= 1ull << j;
            }
            p.tile_mask[static_cast<size_t>(st) * kTilesPerSuper + wt] = m;
        }
    }
    if (p.super_order == nullptr) return;
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence(); // this block's counts are visible before its ticket
        last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // (band_rows > 0 -- a banded order -- implies one rank: super-tile st is screen super-tile st)
    order_by_count(count, gridDim.x, const_cast<uint32_t*>(p.super_order), p.n_super_x, p.band_rows);
    if (threadIdx.x == 0) *done = 0; // ready for the next frame
}

} // namespace vxa
