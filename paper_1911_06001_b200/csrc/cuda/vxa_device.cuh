// Device-side data layout and the per-ray pipeline of the voxanim-b200 frame.
//
// One template serves two instantiations:
//   Real = double : the parity kernel. Compiled with -fmad=false and written in
//                   the reference's operand order, it reproduces the CPU
//                   renderer bit for bit (ray generation renderer.cpp:11-23,
//                   sphere test :25-43, candidate order :134-141,171-203,
//                   trace_ray :63-100, shade :102-113, traversal
//                   traversal.cpp:30-245).
//   Real = float  : the production kernel. Same decision structure (mirror
//                   mask, midpoint recurrence, strict-comparison tie rules,
//                   skip-not-break, nearest (t, id)), FP32 arithmetic, with the
//                   per-instance constants (local ray origin, slab plane
//                   offsets, camera-to-local rotation) folded on the host in
//                   FP64 so each frame's FP32 inputs are rounded once.
//
// HBM layout of a model (built by the upload kernel in vxa_abi.cu, node
// numbering identical to SvoModel::nodes):
//   words : uint2 per node  {x = valid | leaf << 8 | kMixed, y = base}
//           base = child_base when the node has internal children, else
//           attr_base; kMixed marks the rare node with both kinds, whose
//           attr_base then lives in side[child_base] (child_base is unique
//           among nodes with internal children).
//   attrs : uint32 RGBA8 per attribute.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace vxa {

constexpr uint32_t kMaxDepth = 16;
constexpr uint32_t kExit = 8;
constexpr uint32_t kMixed = 1u << 16;

// Work decomposition: 8x4-pixel warp tiles inside 64x64 super-tiles; super-tiles
// are the unit of the multi-GPU screen partition.
#ifndef VXA_TILE_W
#define VXA_TILE_W 8
#endif
constexpr int kTileW = VXA_TILE_W, kTileH = 32 / VXA_TILE_W;
constexpr int kSuper = 64;
constexpr int kTilesPerSuper = (kSuper / kTileW) * (kSuper / kTileH); // 128
// Work-queue order of the super-tiles when the culling pre-pass runs: longest
// first by candidate count (1) or screen order (0); DESIGN.md §7.
#ifndef VXA_LPT
#define VXA_LPT 1
#endif
// Scenes with more instances than this get the per-super-tile culling pre-pass.
#ifndef VXA_SUPER_MIN
#define VXA_SUPER_MIN 32
#endif
constexpr uint32_t kSuperCullMin = VXA_SUPER_MIN;
// The culling pre-pass also writes per-tile candidate masks (1) or the frame
// kernel tests each tile's cone itself (0).
#ifndef VXA_TILE_MASKS
#define VXA_TILE_MASKS 1
#endif
constexpr uint32_t kSuperCap = 1024; // super-tile list capacity (overflow: scan all)

// Screen partition: 64x64 super-tile s = (y / 64) * n_super_x + x / 64 belongs
// to rank s % world. The frame kernel enumerates a rank's super-tiles as
// s = j * world + rank, which is this map inverted.
__host__ __device__ inline uint32_t super_tiles_x(int32_t width) { return static_cast<uint32_t>((width + kSuper - 1) / kSuper); }
__host__ __device__ inline int32_t tile_owner(int32_t x, int32_t y, int32_t width, int32_t world) {
    const uint32_t s = static_cast<uint32_t>(y / kSuper) * super_tiles_x(width) + static_cast<uint32_t>(x / kSuper);
    return static_cast<int32_t>(s % static_cast<uint32_t>(world));
}

struct DevModel {
    const uint2* words;     // general 8-byte node words
    const uint32_t* side;   // attr_base of mixed nodes, indexed by child_base
    const uint32_t* cwords; // compact 4-byte words (canonical models only) or null
    const uint32_t* attrs;
    uint32_t depth;
    uint32_t node_count;
    // Squared radius (unit-cube coordinates, about the cube centre, margin
    // included) of a sphere holding every leaf (vxa_abi.cu: content_radius);
    // >= 0.75 when it is no tighter than the cube's own corners.
    float content_r2;
    uint32_t pad;
};

// (FrameParams::top_words: the model whose first VXA_SMEM_TOP node words the
// frame kernel stages in shared memory, when every instance uses it.)

// Node word policies of the FP32 core.
// WideNodes: {valid | leaf << 8 | mixed, base} for any valid model.
// CompactNodes: valid | base << 8 (base < 2^24), for canonical models -- leaves
// exactly at the last level, none above it (every model build_from_grid or the
// procedural builder produces): the leaf mask is implied by the level, halving
// the node bytes the traversal touches.
struct WideNodes {
    const uint2* w;
    const uint32_t* side;
    using Word = uint2;
    static constexpr bool kLastLevelLeaves = false;
    __device__ __forceinline__ Word load(uint32_t i) const { return __ldg(w + i); }
    __device__ __forceinline__ static uint32_t valid(Word x) { return x.x & 0xffu; }
    __device__ __forceinline__ static uint32_t leaves(Word x, int /*level*/, int /*depth*/) { return (x.x >> 8) & 0xffu; }
    __device__ __forceinline__ static uint32_t child_base(Word x) { return x.y; }
    __device__ __forceinline__ uint32_t attr_base(Word x) const { return (x.x & kMixed) ? __ldg(side + x.y) : x.y; }
    __device__ __forceinline__ static uint2 pack(Word x, uint32_t cur) { return make_uint2(x.x | (cur << 24), x.y); }
    __device__ __forceinline__ static Word unpack(uint2 v, uint32_t& cur) {
        cur = (v.x >> 24) & 0xfu;
        return make_uint2(v.x & 0x00ffffffu, v.y);
    }
};

// Node words staged in shared memory (build variant VXA_SMEM_TOP = words):
// the first top_n words of the scene's model (BFS order: its top levels).
#ifndef VXA_SMEM_TOP
#define VXA_SMEM_TOP 0
#endif
// FP32 core for rays without a zero direction component: position-space planes
// (traverse_pos, 1) or the cell-index planes of traverse_fast (0); DESIGN.md §7.
#ifndef VXA_POSLOOP
#define VXA_POSLOOP 1
#endif
// first_node's octant from the sign bits of tm - t_enter (FMA pipe + shifts;
// 2.8 % faster than three compares and selects on the ALU pipe)
// Stack entries of traverse_pos carry the saved next child's entry parameter
// (16-byte entries), so a pop needs no near planes (-3.7 %).
#ifndef VXA_STACK_TEN
#define VXA_STACK_TEN 1
#endif
// Shared-memory layout of those entries: 0 = 16-byte entries read as 8 + 4 bytes,
// 2 = an 8-byte and a 4-byte array (12 bytes per level and thread: less shared
// memory, more L1).
#ifndef VXA_STACK_LAYOUT
#define VXA_STACK_LAYOUT 2
#endif
#ifndef VXA_FC_SIGN
#define VXA_FC_SIGN 1
#endif
// FP64 parity kernel: rays without a zero local direction component take a
// traverse_model instantiation without the zero-direction midplane convention
#ifndef VXA_F64_SPLIT
#define VXA_F64_SPLIT 1
#endif

// Octant of the first child (first_node, traversal.cpp:63-86): bit a iff the
// midplane is crossed before the entry, tm[a] < te. The sign of the rounded
// difference tm - te is the sign of the exact one (and +0 when equal), so the
// bits can be taken from it.
__device__ __forceinline__ uint32_t first_octant(const float tm[3], float te) {
    if constexpr (VXA_FC_SIGN) {
        const uint32_t x = __float_as_uint(__fsub_rn(tm[0], te)), y = __float_as_uint(__fsub_rn(tm[1], te)),
                       z = __float_as_uint(__fsub_rn(tm[2], te));
        return ((x >> 29) & 4u) | ((y >> 30) & 2u) | (z >> 31);
    } else {
        return (tm[0] < te ? 4u : 0u) | (tm[1] < te ? 2u : 0u) | (tm[2] < te ? 1u : 0u);
    }
}

struct CompactNodes {
    const uint32_t* w;
    uint32_t top_base = 0; // shared address of the staged words (VXA_SMEM_TOP builds)
    uint32_t top_n = 0;    // words staged for this model (0: none)
    using Word = uint32_t;
    static constexpr bool kLastLevelLeaves = true; // leaves exist on the last level only
    __device__ __forceinline__ Word load(uint32_t i) const {
        if constexpr (VXA_SMEM_TOP > 0) {
            if (i < top_n) {
                uint32_t v;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(top_base + 4u * i));
                return v;
            }
        }
        return __ldg(w + i);
    }
    __device__ __forceinline__ static uint32_t valid(Word x) { return x & 0xffu; }
    __device__ __forceinline__ static uint32_t leaves(Word x, int level, int depth) {
        return level + 1 == depth ? (x & 0xffu) : 0u;
    }
    __device__ __forceinline__ static uint32_t child_base(Word x) { return x >> 8; }
    __device__ __forceinline__ uint32_t attr_base(Word x) const { return x >> 8; }
    __device__ __forceinline__ static uint2 pack(Word x, uint32_t cur) { return make_uint2(x, cur); }
    __device__ __forceinline__ static Word unpack(uint2 v, uint32_t& cur) {
        cur = v.y;
        return v.x;
    }
};

// Per-instance frame constants, rebuilt on the host every frame from the FP64
// RigidTransform + Camera (vxa_abi.cu: build_instances).
template <typename Real> struct DevInstance {
    DevModel model;
    Real L[3];    // sphere centre - camera position
    Real L2;      // |L|^2 (reference: l.norm2())
    Real r, r2;   // radius, radius^2
    Real M[9];    // FP64: R^T (world -> local); FP32: R^T C (camera -> local)
    Real R[9];    // world rotation (FP64 normal = R n_local)
    Real A_lo[3]; // -h - o_local  (o_local = R^T (cam - t), FP64)
    Real A_hi[3]; //  h - o_local
    Real h2[3];   // 2h (root cell size)
    float U_lo[3], U_hi[3];   // FP32 kernel: (-h - o) / 2h, (h - o) / 2h (unit-cube plane offsets)
    float Ur_lo[3], Ur_hi[3]; // and their FP64 rounding residuals
    double Md[9]; // FP64 R^T C (camera -> local), FP32 kernel's local direction
    double ih2[3]; // 1 / 2h: local direction -> unit-cube direction (content-sphere test)
    uint32_t zbits[3]; // zero-direction path: bit L set iff o >= centre at level L
    uint32_t zflags;   // bit a: (-h > o); bit 3+a: (h > o)   (zero-direction slab signs)
    int32_t id;
    uint32_t dirty;
    uint32_t valid_model;
    uint32_t pad;
};

template <typename Real> struct FrameParams {
    const DevInstance<Real>* inst;
    // FP32 culling data, one float4 {L (sphere centre - camera), r} per
    // instance (16 B, coalesced and L1-friendly: the cone and sphere tests read
    // only this, not the 300-byte instance records)
    const float4* cull;
    // Large scenes (n_inst > kSuperCullMin): per-super-tile candidate lists
    // from the pre-pass (super_cull_kernel), super_cap entries per rank-local
    // super-tile in instance order; count 0xffffffff = overflow (scan all).
    const uint16_t* super_list;
    const uint32_t* super_count;
    uint32_t super_cap;
    // per 8x4 tile (super-tile major, kTilesPerSuper per super-tile): bit j = entry j of
    // its super-tile's list meets the tile's cone; written by the pre-pass when the list
    // has at most 64 entries (null: the frame kernel tests the cones itself)
    unsigned long long* tile_mask;
    // Processing order of the rank-local super-tiles (super_cull_kernel's last block: most
    // candidates first, so the grid's tail is cheap tiles), or null: natural order.
    const uint32_t* super_order;
    const uint32_t* top_words; // compact words of the scene's single model, or null
    uint32_t top_n;            // words to stage (<= VXA_SMEM_TOP and the model size, multiple of 4)
    uint32_t n_inst;
    int32_t width, height;
    // camera
    Real cam_pos[3];
    Real C[9];         // camera orientation (row-major)
    Real tan_half;     // std::tan(fov * pi / 360), host-evaluated
    Real aspect;       // (double)W / H
    Real inv_w2, inv_h2; // FP32 ray setup: 2/W, 2/H
    Real sx, sy;       // FP32 ray setup: tan_half * aspect, tan_half
    double d_kx, d_ky; // tan_half * aspect / W, tan_half / H in FP64 (FP32 kernel's camera directions)
    uint32_t background; // RGBA8
    uint32_t culling, sorting, sphere_pass;
    uint32_t camera_dirty;
    // partition
    int32_t rank, world;
    uint32_t n_super_x;
    uint32_t super_x_magic; // ceil(2^32 / n_super_x): s / n_super_x = umulhi(s, magic) for s < 2^16
    uint32_t n_tiles; // warp tiles owned by this rank
    uint32_t max_depth; // deepest model of the frame (FP32 shared-memory stack height)
    uint32_t compact;   // every model has compact 4-byte words (FP32 kernel)
    uint32_t fence_sys; // fb is another GPU's framebuffer: every thread fences its stores at system scope
    // outputs
    uint32_t* fb;                 // RGBA8 framebuffer (local or peer-mapped)
    uint8_t* rgb;                 // streamed frames: RGB8 copy for the readback (or null)
    uint32_t* tile_counter;       // persistent-thread work counter
    // Synchronous readback (vxa_render): warp tiles finished per band of
    // band_rows super-tile rows, so the copy engine can start a band's D2H while
    // the frame kernel works on the next ones (null: off)
    uint32_t* band_done;
    uint32_t band_rows;
    // Synchronous readback into page-locked host memory (vxa_render, direct mode):
    // warp tiles finished per super-tile; the warp finishing a super-tile's last
    // tile stores its RGB8 rows into rgb_host (the caller's image, mapped) over
    // PCIe while the frame goes on (null: off)
    uint32_t* super_done;
    uint8_t* rgb_host;
    unsigned long long* counters; // rays, sphere_tests, traversals, reused, fetches, leaf_hits
    uint32_t reset_stats;         // the culling pre-pass zeroes counters (and always tile_counter)
    void* aov;                    // vxa_pixel_aov* or null
    void* hbo;                    // vxa_hit_record* (device copy) or HitRec16* (hbo_compact), or null
    uint32_t hbo_compact;         // FP32 device hit buffer in the 16-byte format
};

// Host-layout records written by the kernel (match include/vxa.h).
struct PixelAov {
    double t;
    int32_t object_id;
    uint32_t node_index;
    uint32_t attr_index;
    uint32_t voxel[3];
    uint8_t level;
    uint8_t kind;
    uint8_t entry_axis;
    uint8_t pad0;
    uint32_t traversals;
    uint32_t node_fetches;
    uint32_t pad1;
};
static_assert(sizeof(PixelAov) == 48, "vxa_pixel_aov layout");

struct HitRec {
    uint32_t color;
    uint32_t pad0;
    double normal[3];
    double t;
    int32_t object_id;
    uint8_t kind;
    uint8_t pad1[3];
};
static_assert(sizeof(HitRec) == 48, "voxanim::HitRecord layout");

// Compact device hit-buffer record of the FP32 kernel (vxa_hbo_create buffers):
// 16 B instead of 48. The world normal is not stored: a record is reused only
// for the same object while it is not dirty, so its normal is the object's
// current R times the stored local normal (entry axis, sign) -- exactly what a
// fresh trace of the same hit computes. Expanded to HitRec on download.
struct HitRec16 {
    uint32_t color;
    float t;
    int32_t object_id;
    uint32_t meta; // kind (bits 0-1) | entry axis << 2 | (local direction positive on it) << 4
};
static_assert(sizeof(HitRec16) == 16, "compact hit record");

// ---------------------------------------------------------------------------
// Node access

__device__ __forceinline__ uint2 load_node(const DevModel& m, uint32_t idx) { return __ldg(m.words + idx); }

__device__ __forceinline__ uint32_t popc8_below(uint32_t mask, uint32_t bit) { return __popc(mask & (bit - 1u)); }

// ---------------------------------------------------------------------------
// Traversal core: Revelles parametric traversal, iterative, explicit stack.
// Follows proj/src/traversal.cpp:115-245 decision for decision.

template <typename Real> struct LocalRay {
    Real d[3];       // unmirrored local direction
    Real t0[3], t1[3]; // root slab parameters of the mirrored ray
    uint32_t mirror; // octant bits of mirrored axes
    uint32_t zero;   // octant bits of zero-direction axes
    uint32_t zbits[3];
};

template <typename Real> struct TravHit {
    Real t;              // max(t_enter, 0)
    Real t_enter_root, t_exit_root;
    uint32_t attr;       // attribute index
    uint32_t parent;     // node index of the leaf's parent
    uint32_t level;      // path_len
    uint32_t axis;       // entry axis
    unsigned long long path; // octant per level, 4 bits each
    uint32_t fetches;
};

__device__ __forceinline__ uint32_t axis_bit(int a) { return 4u >> a; } // x=4, y=2, z=1

template <typename Real> __device__ __forceinline__ Real pos_inf() {
    if constexpr (sizeof(Real) == 8)
        return __longlong_as_double(0x7ff0000000000000ll);
    else
        return __int_as_float(0x7f800000);
}

// Root slab (traversal.cpp:30-61) from host-folded plane offsets:
// unmirrored t0 = A_lo / d, t1 = A_hi / d; a mirrored axis (d < 0) swaps
// them, which is bit-identical to the reference's (-h - (-o)) / (-d) form.
template <typename Real>
__device__ __forceinline__ void setup_root(LocalRay<Real>& r, const Real A_lo[3], const Real A_hi[3],
                                           uint32_t zflags, const uint32_t zbits[3]) {
    const Real inf = pos_inf<Real>();
    r.mirror = 0;
    r.zero = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r.zbits[a] = zbits[a];
        const Real d = r.d[a];
        if (d < Real(0)) r.mirror |= axis_bit(a);
        if (d == Real(0)) {
            r.zero |= axis_bit(a);
            r.t0[a] = (zflags >> a) & 1u ? inf : -inf;
            r.t1[a] = (zflags >> (3 + a)) & 1u ? inf : -inf;
        } else if (d < Real(0)) {
            r.t0[a] = A_hi[a] / d;
            r.t1[a] = A_lo[a] / d;
        } else {
            r.t0[a] = A_lo[a] / d;
            r.t1[a] = A_hi[a] / d;
        }
    }
}

template <typename Real>
__device__ __forceinline__ Real midplane(const LocalRay<Real>& r, int a, const Real t0, const Real t1, int level) {
    if (r.zero & axis_bit(a)) return ((r.zbits[a] >> level) & 1u) ? -pos_inf<Real>() : pos_inf<Real>();
    return Real(0.5) * (t0 + t1);
}

// first_node (traversal.cpp:63-86): octant bit set iff the midplane was crossed
// before the entry parameter.
template <typename Real>
__device__ __forceinline__ uint32_t first_child(const Real t0[3], const Real tm[3]) {
    Real te = t0[0];
    if (t0[1] > te) te = t0[1];
    if (t0[2] > te) te = t0[2];
    uint32_t q = 0;
    if (tm[0] < te) q |= 4u;
    if (tm[1] < te) q |= 2u;
    if (tm[2] < te) q |= 1u;
    return q;
}

// FP32 core: the entry value as one 3-way max (plane parameters are never NaN).
__device__ __forceinline__ uint32_t first_child(const float t0[3], const float tm[3]) {
    const float te = fmaxf(fmaxf(t0[0], t0[1]), t0[2]);
    return (tm[0] < te ? 4u : 0u) | (tm[1] < te ? 2u : 0u) | (tm[2] < te ? 1u : 0u);
}

// next_node (traversal.cpp:88-103): exit axis = argmin t1 (strict <, x first).
template <typename Real> __device__ __forceinline__ uint32_t next_child(const Real t1[3], uint32_t q) {
    uint32_t bit = 4u;
    Real tx = t1[0];
    if (t1[1] < tx) {
        bit = 2u;
        tx = t1[1];
    }
    if (t1[2] < tx) bit = 1u;
    return (q & bit) ? kExit : (q | bit);
}

struct NoLog {
    __device__ __forceinline__ void visit(double, uint32_t, bool) {}
};

// Returns true on a hit. The stack holds the ancestors of the current frame;
// the current frame lives in registers, with its midplane parameters computed
// once when it becomes the frame (push or pop) instead of at every child step
// -- the same 0.5 (t0 + t1) of the same operands, so the same values. kZero =
// false: the caller guarantees no zero direction component (r.zero == 0), so
// the zero-direction midplane convention compiles out (VXA_F64_SPLIT).
template <typename Real, class Log, bool kZero = true>
__device__ bool traverse_model(const DevModel& m, const LocalRay<Real>& r, TravHit<Real>& out, Log& log) {
    Real te = r.t0[0];
    if (r.t0[1] > te) te = r.t0[1];
    if (r.t0[2] > te) te = r.t0[2];
    Real tx = r.t1[0];
    if (r.t1[1] < tx) tx = r.t1[1];
    if (r.t1[2] < tx) tx = r.t1[2];
    out.fetches = 0;
    if (te >= tx || tx < Real(0)) return false;
    out.t_enter_root = te;
    out.t_exit_root = tx;

    Real st0[kMaxDepth][3], st1[kMaxDepth][3];
    uint2 sw[kMaxDepth];
    uint32_t sidx[kMaxDepth], scur[kMaxDepth];

    const auto mid = [&](int a, Real t0, Real t1, int lv) {
        if constexpr (kZero) return midplane(r, a, t0, t1, lv);
        else return Real(0.5) * (t0 + t1);
    };
    Real f0[3] = {r.t0[0], r.t0[1], r.t0[2]};
    Real f1[3] = {r.t1[0], r.t1[1], r.t1[2]};
    Real fm[3]; // the frame's midplane parameters (traversal.cpp:139,167)
    uint32_t fidx = 0;
    uint2 fw = load_node(m, 0);
    uint32_t fetches = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) fm[a] = mid(a, f0[a], f1[a], 0);
    uint32_t fcur = first_child(f0, fm);
    int level = 0;
    unsigned long long path = 0;
    const int depth = static_cast<int>(m.depth);
    // bit L: the frame saved at level L has children left (only those are
    // saved). Popping straight to the deepest one skips exhausted ancestors,
    // which the reference pops one by one with no other effect, and its saved
    // next child is stepped in the same iteration (fall through) -- the same
    // visits in the same order, fewer loop iterations (cf. traverse_fast).
    uint32_t live = 0;

    while (true) {
        if (fcur == kExit) {
            if (live == 0) break;
            asm("bfind.u32 %0, %1;" : "=r"(level) : "r"(live));
            live ^= 1u << level;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                f0[a] = st0[level][a];
                f1[a] = st1[level][a];
                fm[a] = mid(a, f0[a], f1[a], level);
            }
            fw = sw[level];
            fidx = sidx[level];
            fcur = scur[level];
        }
        const uint32_t q = fcur;
        Real c0[3], c1[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (q & axis_bit(a)) {
                c0[a] = fm[a];
                c1[a] = f1[a];
            } else {
                c0[a] = f0[a];
                c1[a] = fm[a];
            }
        }
        fcur = next_child(c1, q);
        // entry parameter = max c0 (the entry axis, argmax with ties to the lower
        // axis, only matters on a hit: taken there)
        Real t_enter = c0[0];
        if (c0[1] > t_enter) t_enter = c0[1];
        if (c0[2] > t_enter) t_enter = c0[2];
        Real t_exit = c1[0];
        if (c1[1] < t_exit) t_exit = c1[1];
        if (c1[2] < t_exit) t_exit = c1[2];
        if (!(t_enter < t_exit) || t_exit < Real(0)) continue;

        const uint32_t oct = q ^ r.mirror;
        const uint32_t bit = 1u << oct;
        const uint32_t valid = fw.x & 0xffu;
        const uint32_t leafm = (fw.x >> 8) & 0xffu;
        if (!(valid & bit)) continue;
        const bool is_leaf = (leafm & bit) != 0;
        log.visit(static_cast<double>(t_enter), static_cast<uint32_t>(level + 1), is_leaf);
        path = (path & ~(0xfull << (4 * level))) | (static_cast<unsigned long long>(oct) << (4 * level));
        if (is_leaf) {
            int entry = 0; // traversal.cpp:214-222
            Real te = c0[0];
            if (c0[1] > te) {
                entry = 1;
                te = c0[1];
            }
            if (c0[2] > te) entry = 2;
            const uint32_t abase = (fw.x & kMixed) ? __ldg(m.side + fw.y) : fw.y;
            out.attr = abase + popc8_below(valid & leafm, bit);
            out.t = t_enter < Real(0) ? Real(0) : t_enter;
            out.parent = fidx;
            out.level = static_cast<uint32_t>(level + 1);
            out.axis = static_cast<uint32_t>(entry);
            out.path = path;
            out.fetches = fetches;
            return true;
        }
        if (level + 1 >= depth || level + 1 >= static_cast<int>(kMaxDepth)) continue;
        const uint32_t child = fw.y + popc8_below(valid & ~leafm, bit);
        // push the current frame (only while it has children left), descend
        if (fcur != kExit) {
            live |= 1u << level;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                st0[level][a] = f0[a];
                st1[level][a] = f1[a];
            }
            sw[level] = fw;
            sidx[level] = fidx;
            scur[level] = fcur;
        }
        ++level;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            f0[a] = c0[a];
            f1[a] = c1[a];
            fm[a] = mid(a, f0[a], f1[a], level);
        }
        fidx = child;
        fw = load_node(m, child);
        ++fetches;
        fcur = first_child(f0, fm);
    }
    out.fetches = fetches;
    return false;
}

// ---------------------------------------------------------------------------
// Production FP32 core: the same Revelles decision structure (mirror mask,
// first_node / next_node with strict comparisons, front-to-back children,
// cull rule, leaf/push rules) but the node's slab planes are derived in
// position space, as the paper does by halving the parent's edge vectors:
// node (c, L) spans [c s_L, (c+1) s_L) of the mirrored axis (s_L = 2h / 2^L,
// halving is exact), and a plane's parameter is t = fma(i, s_L, A) * inv_d
// with A = -h - o (FP64-folded, rounded once). Every plane therefore has one
// t value at every level (siblings share their planes bit for bit: the
// traversal is watertight), the error stays ~2 ulp at any depth, and the
// stack only holds node words: t0/t1/tm are recomputed from the cell
// coordinates on a pop instead of being stored.

struct FastRay {
    // Unit-cube form of each mirrored axis: positions are measured in root
    // cells (x' = (x + h) / 2h), so node planes sit at exact dyadic positions
    // c * 2^-L and the scale 2h only multiplies t (folded into inv).
    // Rays with a zero direction component (traverse_fast<.., true>):
    //   A = (-h - o_m) / 2h rounded, Ar = its FP64 rounding residual times inv.
    // Every other ray (traverse_pos): positions P = 1 + x' in [1, 2] and
    //   A = B = (A_64 - 1) inv rounded once from FP64, so t(P) = fma(P, inv, B); Ar unused.
    float A[3];
    float Ar[3];
    float inv[3]; // 2h / |d|
    // Pruning bound: subtrees entered at t >= t_lim cannot hold a hit that
    // beats the caller's best (t_lim = nextafter(best t), +inf for none).
    float t_lim;
    uint32_t mirror, zero;
    uint32_t zbits[3];
};

struct FastHit {
    float t;
    uint32_t attr, parent, level, axis;
    uint32_t vox[3]; // leaf voxel, unmirrored (leaf_path_to_voxel)
    uint32_t fetches;
};

// t of the plane at position i * sz (i integer-valued, sz = 2^-L) of one
// mirrored axis: X = i * sz + A is exact inside the FMA up to one rounding, and
// t = X * inv + Ari with Ari = A's FP64 rounding residual times inv, one more
// rounding in the second FMA (the residual keeps t accurate when X cancels: a
// plane close to the origin). Every plane gets one value whatever the level
// that computes it, so sibling cells share planes bit for bit (watertight).
__device__ __forceinline__ float plane_t(float i, float sz, float A, float Ari, float inv) {
    return __fmaf_rn(__fmaf_rn(i, sz, A), inv, Ari);
}

__device__ __forceinline__ float zero_mid(const FastRay& r, int a, int level) {
    return ((r.zbits[a] >> level) & 1u) ? -__int_as_float(0x7f800000) : __int_as_float(0x7f800000);
}

__device__ __forceinline__ void fix_zero_axes(const FastRay& r, int level, float t0[3], float tm[3], float t1[3]) {
    const float inf = __int_as_float(0x7f800000);
#pragma unroll
    for (int a = 0; a < 3; ++a)
        if (r.zero & axis_bit(a)) {
            t0[a] = -inf;
            t1[a] = inf;
            tm[a] = zero_mid(r, a, level);
        }
}

// Root setup. d: FP32-rounded local direction; A_lo/A_hi (+ residuals):
// (-h - o) / 2h and (h - o) / 2h folded on the host in FP64; h2 = 2h.
// Returns false when the ray misses the root box (traversal.cpp:56-60).
__device__ __forceinline__ bool fast_setup(FastRay& r, const float d[3], const float A_lo[3], const float A_hi[3],
                                           const float Ar_lo[3], const float Ar_hi[3], const float h2[3],
                                           uint32_t zflags, const uint32_t zbits[3],
                                           float t_lim = __builtin_huge_valf()) {
    r.t_lim = t_lim;
    r.mirror = 0;
    r.zero = 0;
    const float inf = __int_as_float(0x7f800000);
    float te = -inf, tx = inf;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        r.zbits[a] = zbits[a];
        if (d[a] == 0.0f) r.zero |= axis_bit(a);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (d[a] == 0.0f) {
            r.A[a] = 0.0f;
            r.Ar[a] = 0.0f;
            r.inv[a] = 0.0f;
            // zero-direction slab convention: inside iff -h <= o < h
            if ((zflags >> a) & 1u) te = inf;
            if (!((zflags >> (3 + a)) & 1u)) tx = -inf;
        } else {
            const bool m = d[a] < 0.0f;
            if (m) r.mirror |= axis_bit(a);
            const float A = m ? -A_hi[a] : A_lo[a];
            const float Ar = m ? -Ar_hi[a] : Ar_lo[a];
            r.inv[a] = __fdiv_rn(h2[a], fabsf(d[a]));
            if (VXA_POSLOOP && r.zero == 0) {
                // position form: t(P) = fma(P, inv, B), B folded in FP64 and rounded once
                r.A[a] = __double2float_rn(((static_cast<double>(A) - 1.0) + static_cast<double>(Ar)) *
                                           static_cast<double>(r.inv[a]));
                r.Ar[a] = 0.0f;
                te = fmaxf(te, __fmaf_rn(1.0f, r.inv[a], r.A[a]));
                tx = fminf(tx, __fmaf_rn(2.0f, r.inv[a], r.A[a]));
            } else {
                r.A[a] = A;
                r.Ar[a] = __fmul_rn(Ar, r.inv[a]);
                te = fmaxf(te, plane_t(0.0f, 1.0f, r.A[a], r.Ar[a], r.inv[a]));
                tx = fminf(tx, plane_t(1.0f, 1.0f, r.A[a], r.Ar[a], r.inv[a]));
            }
        }
    }
    // a leaf's t is never below its ancestors' entry (shared, monotone planes),
    // so a box entered at or beyond t_lim holds nothing nearer than the best
    return !(te >= tx || tx < 0.0f) && te < t_lim;
}

// Traversal stacks. SmemStack: one column per thread of a [level][thread]
// shared-memory array, addressed through a 32-bit shared-window base kept in
// one register (the compiler otherwise re-derives the generic pointer from
// threadIdx on every push/pop); LocalStack: a private array (API kernel).
template <uint32_t kStride> struct SmemStack {
    uint32_t base; // shared address of this thread's level-0 slot; levels kStride bytes apart
    __device__ __forceinline__ uint2 load(int level) const {
        uint2 v;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(base + level * kStride));
        return v;
    }
    __device__ __forceinline__ void store(int level, uint2 v) const {
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(base + level * kStride), "r"(v.x), "r"(v.y));
    }
    // VXA_STACK_TEN entries: node word, next octant, and that child's entry parameter
#if VXA_STACK_LAYOUT == 2
    // separate [level][thread] arrays: node word + next octant (8 B), entry parameter (4 B)
    uint32_t base_ten;
    __device__ __forceinline__ uint2 load3(int level, float& ten) const {
        uint2 v;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%3];\n\tld.shared.f32 %2, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=f"(ten)
                     : "r"(base + level * kStride), "r"(base_ten + level * (kStride / 2)));
        return v;
    }
    __device__ __forceinline__ void store3(int level, uint2 v, float ten) const {
        asm volatile("st.shared.v2.u32 [%0], {%2, %3};\n\tst.shared.f32 [%1], %4;" ::"r"(base + level * kStride),
                     "r"(base_ten + level * (kStride / 2)), "r"(v.x), "r"(v.y), "f"(ten));
    }
#else
    // 16-byte entries, an 8-byte and a 4-byte access
    __device__ __forceinline__ uint2 load3(int level, float& ten) const {
        uint2 v;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%3];\n\tld.shared.f32 %2, [%3+8];"
                     : "=r"(v.x), "=r"(v.y), "=f"(ten)
                     : "r"(base + level * kStride));
        return v;
    }
    __device__ __forceinline__ void store3(int level, uint2 v, float ten) const {
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n\tst.shared.f32 [%0+8], %3;" ::"r"(base + level * kStride),
                     "r"(v.x), "r"(v.y), "f"(ten));
    }
#endif
};

struct LocalStack {
    uint2 a[kMaxDepth];
    float ten_[kMaxDepth];
    __device__ __forceinline__ uint2 load3(int level, float& ten) const {
        ten = ten_[level];
        return a[level];
    }
    __device__ __forceinline__ void store3(int level, uint2 v, float ten) {
        a[level] = v;
        ten_[level] = ten;
    }
    __device__ __forceinline__ uint2 load(int level) const { return a[level]; }
    __device__ __forceinline__ void store(int level, uint2 v) { a[level] = v; }
};

// Iterative traversal. Every iteration steps one child of the current frame
// (t0/tm/t1 of the node and its cell in registers):
//   * step: the child's exit plane (argmin t1, x first) gives the next octant,
//     or exit -- encoded as fcur >= kExit (q | xb plus 8 xb when the exit
//     axis bit is already set, one integer multiply-add instead of a select);
//   * push: a valid, uncut, internal child becomes the frame. The parent is
//     saved only while it has children left (its word and next octant in the
//     caller's stack column, bit `level` of `live`), so exhausted ancestors
//     are never stored;
//   * pop: when the frame's next is exit, the deepest live ancestor (the
//     highest bit of `live`, bfind) becomes the frame in one jump and its
//     planes are rebuilt from its cell -- a plane's t depends on its position
//     only (plane_t), so the values are the ones the descent computed, bit
//     for bit -- and its saved next child is stepped in the same iteration, so
//     a pop costs its lane no extra iteration (SIMT: fewer iterations for the
//     lanes that pop the most).
// kZero = false: the caller guarantees no zero direction component
// (r.zero == 0), so the zero-direction conventions compile out of the loop.
template <bool kTrackIdx, bool kZero = true, class Nodes, class Stack>
__device__ bool traverse_fast(const Nodes nodes, int model_depth, const FastRay& r, FastHit& out, Stack& stack) {
    uint32_t sidx[kTrackIdx ? kMaxDepth : 1]; // ancestor indices (AOV: leaf parent)
    float c[3] = {1.0f, 1.0f, 1.0f};          // 2 cell + 1: the node's midplane index in half cells (exact)
    float sz = 1.0f;                          // cell size 2^-level
    float t0[3], tm[3], t1[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        t0[a] = plane_t(0.0f, 1.0f, r.A[a], r.Ar[a], r.inv[a]);
        t1[a] = plane_t(1.0f, 1.0f, r.A[a], r.Ar[a], r.inv[a]);
        tm[a] = plane_t(1.0f, 0.5f, r.A[a], r.Ar[a], r.inv[a]);
    }
    if (kZero && r.zero) fix_zero_axes(r, 0, t0, tm, t1);
    typename Nodes::Word fw = nodes.load(0);
    uint32_t fidx = 0, fetches = 1;
    uint32_t fcur = first_child(t0, tm);
    int level = 0;
    const int depth = min(model_depth, static_cast<int>(kMaxDepth));
    uint32_t live = 0; // bit L: the frame saved at level L has children left (only bits < level)

    while (true) {
        if (fcur >= kExit) {
            // pop to the deepest live ancestor
            if (live == 0) break; // every ancestor is exhausted: miss
            int lv;
            asm("bfind.u32 %0, %1;" : "=r"(lv) : "r"(live));
            live ^= 1u << lv;
            fw = Nodes::unpack(stack.load(lv), fcur);
            const float shrink = __int_as_float((127 - (level - lv)) << 23); // 2^-(levels popped)
            level = lv;
            if constexpr (kTrackIdx) fidx = sidx[level];
            sz = __int_as_float((127 - level) << 23); // 2^-level
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                // cell = (c - 1) / 2, ancestor cell = floor(cell * shrink), both exact
                const float hs = 0.5f * shrink;
                const float cn = floorf(__fmaf_rn(c[a], hs, -hs));
                c[a] = __fmaf_rn(2.0f, cn, 1.0f);
                tm[a] = plane_t(c[a], 0.5f * sz, r.A[a], r.Ar[a], r.inv[a]);
                t0[a] = plane_t(cn, sz, r.A[a], r.Ar[a], r.inv[a]);
                t1[a] = plane_t(cn + 1.0f, sz, r.A[a], r.Ar[a], r.inv[a]);
            }
            if (kZero && r.zero) fix_zero_axes(r, level, t0, tm, t1);
            // (falls through: the ancestor's saved next child is stepped now)
        }
        const uint32_t q = fcur;
        float c1[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) c1[a] = (q & axis_bit(a)) ? t1[a] : tm[a];
        // next_node: the exit axis is the first axis attaining min c1 (the
        // strict-< chain's x-first tie rule); the min is also the child's t_exit
        const float t_exit = fminf(fminf(c1[0], c1[1]), c1[2]);
        {
            const uint32_t xb = c1[0] == t_exit ? 4u : (c1[1] == t_exit ? 2u : 1u);
            fcur = (q | xb) + ((q & xb) << 3); // >= kExit iff the exit axis bit is already set
        }
        // An absent child is skipped before its interval is evaluated: the
        // reference culls first and checks node_child second, but both only
        // `continue`, so the order of the two tests is not observable.
        const uint32_t oct = q ^ r.mirror;
        const uint32_t bit = 1u << oct;
        const uint32_t valid = Nodes::valid(fw);
        if (!(valid & bit)) continue;
        float c0[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) c0[a] = (q & axis_bit(a)) ? tm[a] : t0[a];
        // plane parameters are never NaN (finite, or +-inf on zero-direction
        // axes), so max/min equal the reference's compare chains; the entry
        // axis itself is only needed on a hit (below)
        const float t_enter = fmaxf(fmaxf(c0[0], c0[1]), c0[2]);
        // the reference cull !(t_enter < t_exit) || t_exit < 0, plus the pruning
        // bound (t_enter >= t_lim: nothing in this child can beat the best)
        if (!(t_enter < fminf(t_exit, r.t_lim)) || t_exit < 0.0f) continue;
        // compact words: a (valid) child is a leaf exactly on the last level
        bool is_leaf;
        uint32_t leafm;
        if constexpr (Nodes::kLastLevelLeaves) {
            is_leaf = level + 1 == depth;
            leafm = is_leaf ? valid : 0u;
        } else {
            leafm = Nodes::leaves(fw, level, depth);
            is_leaf = (leafm & bit) != 0;
        }
        if (is_leaf) {
            out.attr = nodes.attr_base(fw) + popc8_below(Nodes::kLastLevelLeaves ? valid : valid & leafm, bit);
            out.t = fmaxf(t_enter, 0.0f);
            out.parent = fidx;
            out.level = static_cast<uint32_t>(level + 1);
            // entry axis: argmax of c0, ties to the lower axis (traversal.cpp:214-222)
            uint32_t entry = 0;
            float te = c0[0];
            if (c0[1] > te) entry = 1, te = c0[1];
            if (c0[2] > te) entry = 2;
            out.axis = entry;
            out.fetches = fetches;
            const uint32_t top = (2u << level) - 1u; // 2^(level+1) - 1
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const uint32_t v = static_cast<uint32_t>(c[a]) - 1u + ((q >> (2 - a)) & 1u);
                out.vox[a] = (r.mirror & axis_bit(a)) ? top - v : v;
            }
            return true;
        }
        if constexpr (!Nodes::kLastLevelLeaves) {
            if (level + 1 >= depth) continue;
        }
        // push: save the parent only while it has children left
        const uint32_t child =
            Nodes::child_base(fw) + popc8_below(Nodes::kLastLevelLeaves ? valid : valid & ~leafm, bit);
        if (fcur < kExit) {
            live |= 1u << level;
            stack.store(level, Nodes::pack(fw, fcur));
        }
        if constexpr (kTrackIdx) {
            sidx[level] = fidx;
            fidx = child;
        }
        ++level;
        fw = nodes.load(child);
        ++fetches;
        sz = 0.5f * sz;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            // child midplane index: 2 (2 cell + b) + 1 = 2 c + 2 b - 1
            c[a] = __fmaf_rn(2.0f, c[a], (q & axis_bit(a)) ? 1.0f : -1.0f);
            tm[a] = plane_t(c[a], 0.5f * sz, r.A[a], r.Ar[a], r.inv[a]);
            t0[a] = c0[a];
            t1[a] = c1[a];
        }
        if (kZero && r.zero) {
#pragma unroll
            for (int a = 0; a < 3; ++a)
                if (r.zero & axis_bit(a)) tm[a] = zero_mid(r, a, level);
        }
        fcur = first_child(t0, tm);
    }
    out.fetches = fetches;
    return false;
}

// Position-space FP32 core for rays without a zero direction component (the
// same decisions as traverse_fast, fewer instructions and registers). Each
// mirrored axis is measured in root cells shifted by one, P in [1, 2]: a node
// at level L spans [1 + c 2^-L, 1 + (c + 1) 2^-L), so its low corner is any
// interior position with the mantissa bits below 23 - L cleared and its
// midplane sets bit 22 - L -- a pop rebuilds an ancestor's planes with two
// bit operations per axis (no floor). A plane's parameter is
// t = fma(P, inv, B): one rounding of an exact product plus B (FastRay), so
// every plane still has one value at every level (watertight), and a pop
// reproduces the descent's values bit for bit.
// State: the node's midplane positions pm, midplane and far-plane parameters
// tm / t1 (no near planes: the entry parameter of the child being stepped is
// carried as `ten` -- the next sibling's entry is max(ten, t_exit) exactly,
// because it differs from the current child only on the exit axis, whose near
// plane is below its exit plane), the node word, the next octant, the level
// and the `live` mask of ancestors with children left (level L at bit 22 - L: its midplane bit).
template <bool kTrackIdx, class Nodes, class Stack>
__device__ bool traverse_pos(const Nodes nodes, int model_depth, const FastRay& r, FastHit& out, Stack& stack) {
    uint32_t sidx[kTrackIdx ? kMaxDepth : 1];
    float pm[3], tm[3], t1[3];
    float ten; // entry parameter of the child fcur (first_node: the node's own entry)
    {
        float t0[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            pm[a] = 1.5f;
            t0[a] = __fmaf_rn(1.0f, r.inv[a], r.A[a]);
            tm[a] = __fmaf_rn(1.5f, r.inv[a], r.A[a]);
            t1[a] = __fmaf_rn(2.0f, r.inv[a], r.A[a]);
        }
        ten = fmaxf(fmaxf(t0[0], t0[1]), t0[2]);
    }
    typename Nodes::Word fw = nodes.load(0);
    uint32_t fidx = 0, fetches = 1;
    // first_node: octant bit iff the midplane is crossed before the entry
    uint32_t fcur = first_octant(tm, ten);
    int level = 0;
    const int depth = min(model_depth, static_cast<int>(kMaxDepth));
    uint32_t live = 0;

    while (true) {
        if (fcur >= kExit) {
            // pop to the deepest live ancestor, its planes rebuilt from the position bits
            // `live` holds level L's bit at position 22 - L, which is the level's midplane
            // bit in the position words: the deepest live level is the lowest set bit,
            // and that bit is the `mid` its planes are rebuilt with (-1.8 %)
            const uint32_t mid = live & (0u - live); // 2^-(lv+1) as a mantissa bit
            if (mid == 0) break;                     // every ancestor is exhausted: miss
            live ^= mid;
            int lv;
            asm("bfind.u32 %0, %1;" : "=r"(lv) : "r"(mid));
            lv = 22 - lv;
            const uint32_t keep = 0u - (mid << 1); // sign, exponent and the level-lv cell bits
            if constexpr (VXA_STACK_TEN)
                fw = Nodes::unpack(stack.load3(lv, ten), fcur); // with the saved next child's entry
            else
                fw = Nodes::unpack(stack.load(lv), fcur);
            level = lv;
            if constexpr (kTrackIdx) fidx = sidx[level];
            const float half = __int_as_float((126 - lv) << 23); // the value of `mid`
            const uint32_t q = fcur;
            float c0[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const float lo = __uint_as_float(__float_as_uint(pm[a]) & keep);
                pm[a] = __uint_as_float(__float_as_uint(lo) | mid);
                tm[a] = __fmaf_rn(pm[a], r.inv[a], r.A[a]);
                t1[a] = __fmaf_rn(pm[a] + half, r.inv[a], r.A[a]); // far plane: pm + half = lo + size, exact
                if constexpr (!VXA_STACK_TEN) c0[a] = (q & axis_bit(a)) ? tm[a] : __fmaf_rn(lo, r.inv[a], r.A[a]);
            }
            if constexpr (!VXA_STACK_TEN) ten = fmaxf(fmaxf(c0[0], c0[1]), c0[2]); // entry of the saved next child
            // (falls through: the ancestor's saved next child is stepped now)
        }
        const uint32_t q = fcur;
        float c1[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) c1[a] = (q & axis_bit(a)) ? t1[a] : tm[a];
        // next_node: the exit axis is the first axis attaining min c1 (x first)
        const float t_exit = fminf(fminf(c1[0], c1[1]), c1[2]);
        {
            const uint32_t xb = c1[0] == t_exit ? 4u : (c1[1] == t_exit ? 2u : 1u);
            // (q | xb) + 8 (q & xb), >= kExit iff the exit axis bit is already set; as
            // q + xb + 7 (q & xb) the multiply-add runs on the FMA pipe (the ALU pipe is
            // the loop's busiest: -0.5 %)
            fcur = q + xb + 7u * (q & xb);
        }
        const float t_enter = ten;
        ten = fmaxf(ten, t_exit);
        const uint32_t oct = q ^ r.mirror;
        const uint32_t bit = 1u << oct;
        const uint32_t valid = Nodes::valid(fw);
        if (!(valid & bit)) continue;
        if (!(t_enter < fminf(t_exit, r.t_lim)) || t_exit < 0.0f) continue;
        bool is_leaf;
        uint32_t leafm;
        if constexpr (Nodes::kLastLevelLeaves) {
            is_leaf = level + 1 == depth;
            leafm = is_leaf ? valid : 0u;
        } else {
            leafm = Nodes::leaves(fw, level, depth);
            is_leaf = (leafm & bit) != 0;
        }
        if (is_leaf) {
            out.attr = nodes.attr_base(fw) + popc8_below(Nodes::kLastLevelLeaves ? valid : valid & leafm, bit);
            out.t = fmaxf(t_enter, 0.0f);
            out.parent = fidx;
            out.level = static_cast<uint32_t>(level + 1);
            // entry axis: argmax of the child's near planes, ties to the lower axis
            // (traversal.cpp:214-222); the node's near planes from its low corner
            const uint32_t keep = 0xffffffffu << (23 - level);
            float c0[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const float lo = __uint_as_float(__float_as_uint(pm[a]) & keep);
                c0[a] = (q & axis_bit(a)) ? tm[a] : __fmaf_rn(lo, r.inv[a], r.A[a]);
            }
            uint32_t entry = 0;
            float te = c0[0];
            if (c0[1] > te) entry = 1, te = c0[1];
            if (c0[2] > te) entry = 2;
            out.axis = entry;
            out.fetches = fetches;
            const uint32_t top = (2u << level) - 1u; // 2^(level+1) - 1
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const uint32_t cell = (__float_as_uint(pm[a]) & 0x7fffffu) >> (23 - level);
                const uint32_t v = 2u * cell + ((q >> (2 - a)) & 1u);
                out.vox[a] = (r.mirror & axis_bit(a)) ? top - v : v;
            }
            return true;
        }
        if constexpr (!Nodes::kLastLevelLeaves) {
            if (level + 1 >= depth) continue;
        }
        // push: save the parent only while it has children left
        const uint32_t child =
            Nodes::child_base(fw) + popc8_below(Nodes::kLastLevelLeaves ? valid : valid & ~leafm, bit);
        if (fcur < kExit) {
            live |= 0x400000u >> level; // level L at bit 22 - L (the pop above)
            if constexpr (VXA_STACK_TEN)
                stack.store3(level, Nodes::pack(fw, fcur), ten); // ten = the next sibling's entry here
            else
                stack.store(level, Nodes::pack(fw, fcur));
        }
        if constexpr (kTrackIdx) {
            sidx[level] = fidx;
            fidx = child;
        }
        const float quarter = __int_as_float((125 - level) << 23); // 2^-(level+2): child half-size
        ++level;
        fw = nodes.load(child);
        ++fetches;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            // child midplane: +- a quarter of the node (exact), picked by the octant bit
            // (a select of +-quarter and an add: no +-1 constant, -1.3 %)
            pm[a] = __fadd_rn(pm[a], (q & axis_bit(a)) ? quarter : -quarter);
            tm[a] = __fmaf_rn(pm[a], r.inv[a], r.A[a]);
            t1[a] = c1[a];
        }
        ten = t_enter; // the child's entry = its first child's entry
        fcur = first_octant(tm, ten);
    }
    out.fetches = fetches;
    return false;
}

// Voxel coordinates of a hit path (leaf_path_to_voxel, traversal.cpp:260-268).
__device__ __forceinline__ void path_to_voxel(unsigned long long path, uint32_t len, uint32_t v[3]) {
    v[0] = v[1] = v[2] = 0;
    for (uint32_t l = 0; l < len; ++l) {
        const uint32_t o = static_cast<uint32_t>(path >> (4 * l)) & 0xfu;
        v[0] = (v[0] << 1) | ((o >> 2) & 1u);
        v[1] = (v[1] << 1) | ((o >> 1) & 1u);
        v[2] = (v[2] << 1) | (o & 1u);
    }
}

} // namespace vxa
