// Device SVO builder: the reference's build_from_grid (proj/src/svo.cpp:52-132)
// from a dense occupancy grid (VoxelGrid bitset, proj/include/voxanim/ingest.hpp:34-63)
// straight into device memory, SURVEY.md §8(f) rank 2.
//
// The reference recurses over all 8^depth sub-cubes into a pointer tree and
// linearises it FIFO: per popped node, octants 0..7 in order, leaves append an
// attribute, internal children are enqueued (svo.cpp:100-131). FIFO over a
// tree whose children are visited in octant order numbers every level in
// octant-path order, i.e. in Morton order with x the most significant bit of
// each triple (octant_bit_x = 4, svo.hpp:21-23). Hence, with V_L[c] the
// child-occupancy byte of cube c of the 2^L lattice (its valid_mask):
//   node index of an occupied level-L cube = (nodes above level L) + its rank
//       among the occupied level-L cubes in Morton order;
//   child_base = first node of level L+1 + (set bits of V_L before c);
//   attr_base (last level) = set bits of V_{depth-1} before c.
// So the build is: one pass that gathers the grid into V_{depth-1} (Morton
// order), a byte-reduction pyramid up to V_0, one popcount reduction per
// level for the level sizes, then per level an exclusive scan of the child
// counts of the occupied cubes and an emission pass writing the 12-byte
// records, the compact render words, the next level's cube list and, on the
// last level, the attributes (voxel_color, ingest.cpp:24-29,67-85). Every
// pass is a streaming pass over HBM; no pointer tree, no host work.
#include <cub/cub.cuh>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "vxa_internal.h"

namespace vxa {
namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t n) {
    const uint64_t b = (n + kThreads - 1) / kThreads;
    return static_cast<unsigned>(b < 148u * 64u ? (b == 0 ? 1 : b) : 148u * 64u);
}

// every third bit of v (bits 0, 3, 6, ...) packed together
__device__ __forceinline__ uint32_t compact3(uint32_t v) {
    v &= 0x09249249u;
    v = (v ^ (v >> 2)) & 0x030c30c3u;
    v = (v ^ (v >> 4)) & 0x0300f00fu;
    v = (v ^ (v >> 8)) & 0xff0000ffu;
    v = (v ^ (v >> 16)) & 0x000003ffu;
    return v;
}

// Content bound of the built model: the largest squared distance, in unit-cube
// coordinates about the cube centre, of any leaf's farthest corner (the FP32
// frame kernel's content-sphere test, vxa_abi.cu: content_r2), from one byte of
// V_{depth-1} per cube. Exact in FP32: coordinates are multiples of 2^-depth
// (depth <= 10), their squares and sums fit the mantissa. Maximum through the
// float bits (non-negative floats order like unsigned ints).
__global__ void leaf_extent(const uint8_t* __restrict__ v, uint64_t cubes, uint32_t depth,
                            unsigned int* __restrict__ out) {
    const float sz = ldexpf(1.0f, -static_cast<int>(depth));
    float best = 0.0f;
    for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < cubes; i += uint64_t{gridDim.x} * blockDim.x) {
        const uint32_t b = v[i];
        if (b == 0) continue;
        const uint32_t c = static_cast<uint32_t>(i);
        const uint32_t cx = compact3(c >> 2), cy = compact3(c >> 1), cz = compact3(c);
        for (uint32_t o = 0; o < 8; ++o) {
            if (!((b >> o) & 1u)) continue;
            const uint32_t q[3] = {2 * cx + ((o >> 2) & 1u), 2 * cy + ((o >> 1) & 1u), 2 * cz + (o & 1u)};
            float acc = 0.0f;
            for (int a = 0; a < 3; ++a) {
                const float lo = static_cast<float>(q[a]) * sz - 0.5f, hi = static_cast<float>(q[a] + 1) * sz - 0.5f;
                acc += fmaxf(lo * lo, hi * hi);
            }
            best = fmaxf(best, acc);
        }
    }
    for (int d = 16; d > 0; d >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, d));
    if ((threadIdx.x & 31u) == 0 && best > 0.0f) atomicMax(out, __float_as_uint(best));
}

// V_{depth-1}: for each cube c of the 2^(depth-1) lattice, the occupancy of
// its 8 voxels as the octant mask. Voxels (2x+i, 2y+j, 2z..2z+1) are two
// adjacent bits of the x-major bitset (bit (x*n + y)*n + z, z even).
__global__ void leaf_masks(const uint64_t* __restrict__ grid, uint32_t n, uint64_t cubes, uint8_t* __restrict__ v) {
    for (uint64_t c = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; c < cubes;
         c += uint64_t{gridDim.x} * blockDim.x) {
        const uint32_t code = static_cast<uint32_t>(c);
        const uint64_t x = compact3(code >> 2), y = compact3(code >> 1), z = compact3(code);
        uint32_t mask = 0;
#pragma unroll
        for (uint32_t i = 0; i < 2; ++i)
#pragma unroll
            for (uint32_t j = 0; j < 2; ++j) {
                const uint64_t b = ((2 * x + i) * n + (2 * y + j)) * n + 2 * z;
                const uint32_t two = static_cast<uint32_t>(__ldg(grid + (b >> 6)) >> (b & 63)) & 3u;
                mask |= two << (4 * i + 2 * j); // octant (i<<2)|(j<<1)|k, k = bit
            }
        v[c] = static_cast<uint8_t>(mask);
    }
}

// Four Morton-consecutive cubes 4q..4q+3 per thread (they differ in the
// cube's lowest y and z bits): 2 x-rows x 4 y-rows of 4 z-bits each -- 8 word
// loads and one 32-bit store for 4 cubes instead of 16 loads and 4 byte stores.
__global__ void leaf_masks4(const uint64_t* __restrict__ grid, uint32_t n, uint64_t quads, uint32_t* __restrict__ v) {
    for (uint64_t q = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; q < quads;
         q += uint64_t{gridDim.x} * blockDim.x) {
        const uint32_t code = static_cast<uint32_t>(q) << 2; // cube of the first of the four
        const uint64_t x = compact3(code >> 2), y = compact3(code >> 1), z = compact3(code);
        // voxel rows: x in {2x, 2x+1}, y in {2y .. 2y+3}; z bits 2z .. 2z+3 (2z is a multiple of 4)
        uint32_t nib[2][4];
#pragma unroll
        for (uint32_t i = 0; i < 2; ++i)
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) {
                const uint64_t b = ((2 * x + i) * n + (2 * y + j)) * n + 2 * z;
                nib[i][j] = static_cast<uint32_t>(__ldg(grid + (b >> 6)) >> (b & 63)) & 0xfu;
            }
        uint32_t out = 0;
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) { // cube 4q + k: z0 = k & 1, y0 = k >> 1
            const uint32_t z0 = k & 1u, y0 = k >> 1;
            uint32_t mask = 0;
#pragma unroll
            for (uint32_t i = 0; i < 2; ++i)
#pragma unroll
                for (uint32_t j = 0; j < 2; ++j)
                    mask |= ((nib[i][2 * y0 + j] >> (2 * z0)) & 3u) << (4 * i + 2 * j);
            out |= mask << (8 * k);
        }
        v[q] = out;
    }
}

// V_{L-1}[c] bit o = (V_L[8c + o] != 0)
__global__ void parent_masks(const uint64_t* __restrict__ child, uint64_t cubes, uint8_t* __restrict__ v) {
    for (uint64_t c = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; c < cubes;
         c += uint64_t{gridDim.x} * blockDim.x) {
        const uint64_t w = child[c];
        uint32_t m = 0;
#pragma unroll
        for (int o = 0; o < 8; ++o) m |= ((w >> (8 * o)) & 0xffu) ? (1u << o) : 0u;
        v[c] = static_cast<uint8_t>(m);
    }
}

// total set bits of a byte array (= number of occupied cubes one level down)
__global__ void count_bits(const uint8_t* __restrict__ v, uint64_t bytes, unsigned long long* __restrict__ out) {
    uint32_t s = 0;
    const uint64_t words = bytes / 4;
    const auto* w4 = reinterpret_cast<const uint32_t*>(v);
    for (uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x; i < words; i += uint64_t{gridDim.x} * blockDim.x)
        s += __popc(__ldg(w4 + i));
    if (blockIdx.x == 0 && threadIdx.x < bytes % 4) s += __popc(v[words * 4 + threadIdx.x]);
    using Reduce = cub::BlockReduce<uint32_t, kThreads>;
    __shared__ typename Reduce::TempStorage tmp;
    const uint32_t total = Reduce(tmp).Sum(s);
    if (threadIdx.x == 0 && total) atomicAdd(out, static_cast<unsigned long long>(total));
}

__global__ void child_counts(const uint32_t* __restrict__ codes, uint32_t n, const uint8_t* __restrict__ v,
                             uint32_t* __restrict__ cnt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        cnt[i] = __popc(v[codes[i]]);
}

// voxel_color (ingest.cpp:24-29,67-85): SplitMix64 finaliser of x<<42|y<<21|z,
// or the by-height ramp lround(from + (to - from) * y / (n - 1)) in unfused FP64.
__device__ __forceinline__ uint32_t voxel_color(uint32_t mode, uint32_t constant, uint32_t n, uint32_t x, uint32_t y,
                                                uint32_t z) {
    if (mode == 2) return constant;
    if (mode == 1) {
        const double f = n > 1 ? __ddiv_rn(static_cast<double>(y), static_cast<double>(n - 1)) : 0.0;
        const auto ramp = [f](double from, double to) {
            return static_cast<uint32_t>(lround(__dadd_rn(from, __dmul_rn(__dadd_rn(to, -from), f)))) & 0xffu;
        };
        return ramp(40, 235) | (ramp(90, 170) << 8) | (ramp(200, 60) << 16) | 0xff000000u;
    }
    uint64_t k = (uint64_t{x} << 42) | (uint64_t{y} << 21) | z;
    k += 0x9e3779b97f4a7c15ull;
    k = (k ^ (k >> 30)) * 0xbf58476d1ce4e5b9ull;
    k = (k ^ (k >> 27)) * 0x94d049bb133111ebull;
    k ^= k >> 31;
    return (64u + (k & 0xbfu)) | ((64u + ((k >> 8) & 0xbfu)) << 8) | ((64u + ((k >> 16) & 0xbfu)) << 16) |
           0xff000000u;
}

struct LevelArgs {
    const uint32_t* codes; // occupied cubes of this level, Morton order
    uint32_t n;            // their count
    const uint8_t* v;      // V_L
    const uint32_t* excl;  // exclusive scan of the child counts
    uint32_t first;        // node index of codes[0]
    uint32_t next_first;   // node index of the first node one level down
    bool last;             // children are voxels
    uint32_t* records;     // 12-byte SvoNode records (3 words)
    uint32_t* cwords;      // compact render words, or null
    uint32_t* next_codes;  // cube list of level L+1 (internal levels)
    uint32_t* attrs;       // attributes (last level)
    uint32_t color_mode, color_constant, resolution;
};

__global__ void emit_level(LevelArgs a) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        const uint32_t c = a.codes[i];
        const uint32_t valid = a.v[c];
        const uint32_t e = a.excl[i];
        const uint32_t node = a.first + i;
        uint32_t child_base = 0, attr_base = 0, leaf = 0;
        if (!a.last) {
            if (valid) child_base = a.next_first + e;
        } else {
            leaf = valid;
            if (valid) attr_base = e;
        }
        a.records[3 * size_t{node}] = child_base;
        a.records[3 * size_t{node} + 1] = attr_base;
        a.records[3 * size_t{node} + 2] = valid | (leaf << 8);
        if (a.cwords) a.cwords[node] = valid | ((a.last ? attr_base : child_base) << 8);
        uint32_t r = 0;
        for (uint32_t o = 0; o < 8; ++o) {
            if (!((valid >> o) & 1u)) continue;
            const uint32_t k = 8u * c + o;
            if (!a.last) {
                a.next_codes[e + r] = k;
            } else {
                a.attrs[e + r] = voxel_color(a.color_mode, a.color_constant, a.resolution, compact3(k >> 2),
                                             compact3(k >> 1), compact3(k));
            }
            ++r;
        }
    }
}

// Position of the r-th (0-based) set bit of an 8-bit mask (branch-free).
__device__ __forceinline__ uint32_t nth_set_bit8(uint32_t m, uint32_t r) {
    uint32_t p = 0;
    const uint32_t c4 = __popc(m & 0xfu);
    if (r >= c4) r -= c4, p = 4;
    const uint32_t c2 = __popc((m >> p) & 0x3u);
    if (r >= c2) r -= c2, p += 2;
    return p + (r >= ((m >> p) & 1u) ? 1u : 0u);
}

// The last level (children are voxels), warp-cooperatively: a warp takes 32
// consecutive nodes, whose attributes are one contiguous range of the output
// (the scan). Lane j produces outputs j, j + 32, ... of that range; the node
// of an output is found from the 32-bit map of node starts inside the current
// 32-output chunk (one OR-reduction) plus the count of nodes starting before
// it (one ballot); its octant is the r-th set bit of the node's mask. The
// colour hash runs with every lane busy and the stores are fully coalesced
// (the per-node octant loop of emit_level is divergent and its stores strided).
__global__ void __launch_bounds__(256) emit_leaves(LevelArgs a) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warps = gridDim.x * (blockDim.x / 32u);
    for (uint32_t g = blockIdx.x * (blockDim.x / 32u) + (threadIdx.x >> 5); g * 32u < a.n; g += warps) {
        const uint32_t i = g * 32u + lane;
        const uint32_t n_live = min(32u, a.n - g * 32u);
        const bool live = lane < n_live;
        const uint32_t c = live ? a.codes[i] : 0u;
        const uint32_t valid = live ? a.v[c] : 0u;
        const uint32_t e = live ? a.excl[i] : 0u;
        if (live) {
            const uint32_t node = a.first + i;
            const uint32_t attr_base = valid ? e : 0u;
            a.records[3 * size_t{node}] = 0u;
            a.records[3 * size_t{node} + 1] = attr_base;
            a.records[3 * size_t{node} + 2] = valid | (valid << 8);
            if (a.cwords) a.cwords[node] = valid | (attr_base << 8);
        }
        // the node's cube, 10 bits per axis, voxel = 2 * cube + octant bit
        const uint32_t xyz = (compact3(c >> 2) << 20) | (compact3(c >> 1) << 10) | compact3(c);
        const uint32_t e0 = __shfl_sync(0xffffffffu, e, 0);
        const uint32_t total = __shfl_sync(0xffffffffu, e + __popc(valid), n_live - 1u) - e0;
        const uint32_t rel = e - e0; // this node's first output, relative to e0
        for (uint32_t o0 = 0; o0 < total; o0 += 32u) {
            // every live node has >= 1 voxel, so node starts are distinct
            const bool starts_here = live && rel >= o0 && rel < o0 + 32u;
            const uint32_t starts = __reduce_or_sync(0xffffffffu, starts_here ? 1u << (rel - o0) : 0u);
            const uint32_t before = __popc(__ballot_sync(0xffffffffu, live && rel < o0));
            const uint32_t k = before + __popc(starts & ((2u << lane) - 1u)) - 1u;
            const uint32_t rk = __shfl_sync(0xffffffffu, rel, k);
            const uint32_t vk = __shfl_sync(0xffffffffu, valid, k);
            const uint32_t pk = __shfl_sync(0xffffffffu, xyz, k);
            const uint32_t o = o0 + lane;
            if (o < total) {
                const uint32_t oct = nth_set_bit8(vk, o - rk);
                const uint32_t x = 2u * (pk >> 20) + ((oct >> 2) & 1u);
                const uint32_t y = 2u * ((pk >> 10) & 0x3ffu) + ((oct >> 1) & 1u);
                const uint32_t z = 2u * (pk & 0x3ffu) + (oct & 1u);
                a.attrs[e0 + o] = voxel_color(a.color_mode, a.color_constant, a.resolution, x, y, z);
            }
        }
    }
}

inline size_t align_up(uint64_t b) { return static_cast<size_t>((b + 255) & ~uint64_t{255}); }

} // namespace

// Builds the model of a dense grid already resident on the device (grid_dev:
// (n^3 + 63) / 64 words, n = 2^depth, depth in [1, 10]). On success the caller
// owns out.records / out.attrs / out.cwords (cwords null when the model is too
// large for 24-bit bases).
namespace {
// VOXANIM_BUILD_TRACE=1: per-phase wall clock of build_svo on stderr (synchronising)
struct Trace {
    bool on = std::getenv("VOXANIM_BUILD_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(cudaStream_t s, const char* what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[build] %-12s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};
} // namespace

cudaError_t build_svo(cudaStream_t s, const uint64_t* grid_dev, uint32_t depth, uint32_t color_mode,
                      uint32_t color_constant, BuildScratch& scratch, BuiltModel& out) {
    Trace tr;
    const uint32_t n = 1u << depth;
    // Scratch, phase 1: the V pyramid (V[L]: 8^L bytes, padded to 8 for the
    // 64-bit reads) and the level-size counters, in one grow-only arena.
    std::vector<uint8_t*> V(depth);
    {
        std::vector<size_t> off(depth + 1, 0);
        for (uint32_t L = 0; L < depth; ++L)
            off[L + 1] = off[L] + align_up(std::max<uint64_t>(8, uint64_t{1} << (3 * L)));
        if (cudaError_t e = scratch.pyramid.ensure(off[depth] + 8 * size_t{depth} + 8); e != cudaSuccess) return e;
        for (uint32_t L = 0; L < depth; ++L) V[L] = static_cast<uint8_t*>(scratch.pyramid.p) + off[L];
    }
    auto* counts = reinterpret_cast<unsigned long long*>(V[depth - 1] + align_up(std::max<uint64_t>(
                                                                          8, uint64_t{1} << (3 * (depth - 1)))));
    tr.mark(s, "alloc V");
    const uint64_t top = uint64_t{1} << (3 * (depth - 1));
    if (top % 4 == 0)
        leaf_masks4<<<grid_for(top / 4), kThreads, 0, s>>>(grid_dev, n, top / 4, reinterpret_cast<uint32_t*>(V[depth - 1]));
    else
        leaf_masks<<<grid_for(top), kThreads, 0, s>>>(grid_dev, n, top, V[depth - 1]);
    for (uint32_t L = depth - 1; L >= 1; --L) {
        const uint64_t cubes = uint64_t{1} << (3 * (L - 1));
        parent_masks<<<grid_for(cubes), kThreads, 0, s>>>(reinterpret_cast<const uint64_t*>(V[L]), cubes, V[L - 1]);
    }
    tr.mark(s, "pyramid");
    // level sizes: N_0 = 1 (the root always exists), N_{L+1} = set bits of V_L;
    // then the leaves' extent (content bound) behind them
    cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * depth + 8, s);
    auto* extent = reinterpret_cast<unsigned int*>(counts + depth);
    leaf_extent<<<grid_for(top), kThreads, 0, s>>>(V[depth - 1], top, depth, extent);
    out.extent_dev = extent;
    for (uint32_t L = 0; L < depth; ++L) {
        const uint64_t bytes = uint64_t{1} << (3 * L);
        count_bits<<<grid_for(bytes / 4 + 1), kThreads, 0, s>>>(V[L], bytes, counts + L);
    }
    std::vector<unsigned long long> N(depth + 1, 1);
    if (cudaError_t e =
            cudaMemcpyAsync(N.data() + 1, counts, sizeof(unsigned long long) * depth, cudaMemcpyDeviceToHost, s);
        e != cudaSuccess)
        return e;
    if (cudaError_t e = cudaStreamSynchronize(s); e != cudaSuccess) return e;
    uint64_t nodes = 0, widest = 1;
    for (uint32_t L = 0; L < depth; ++L) {
        nodes += N[L];
        widest = std::max<uint64_t>(widest, N[L]);
    }
    const uint64_t leaves = N[depth];
    if (nodes >= (uint64_t{1} << 32) || leaves >= (uint64_t{1} << 32)) return cudaErrorInvalidValue;
    const bool compact = nodes < (1u << 24) && leaves <= (1u << 24);
    tr.mark(s, "counts");

    // Scratch, phase 2: cube lists (ping-pong), child counts, their scan.
    size_t scan_bytes = 0;
    if (cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, static_cast<uint32_t*>(nullptr),
                                                      static_cast<uint32_t*>(nullptr), static_cast<int>(widest), s);
        e != cudaSuccess)
        return e;
    const size_t list = align_up(4 * widest);
    if (cudaError_t e = scratch.levels.ensure(4 * list + align_up(scan_bytes)); e != cudaSuccess) return e;
    auto* lv = static_cast<uint8_t*>(scratch.levels.p);
    uint32_t* codes_a = reinterpret_cast<uint32_t*>(lv);
    uint32_t* codes_b = reinterpret_cast<uint32_t*>(lv + list);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(lv + 2 * list);
    uint32_t* excl = reinterpret_cast<uint32_t*>(lv + 3 * list);
    void* scan_tmp = lv + 4 * list;

    // The model: one allocation holding the records, attributes, compact and
    // wide render words (owned by the model entry from here on).
    const size_t rec_b = align_up(12 * nodes), attr_b = align_up(4 * std::max<uint64_t>(leaves, 1)),
                 cw_b = compact ? align_up(4 * nodes) : 0, w_b = align_up(8 * nodes);
    void* block = nullptr;
    if (cudaError_t e = cudaMalloc(&block, rec_b + attr_b + cw_b + w_b); e != cudaSuccess) return e;
    auto* bp = static_cast<uint8_t*>(block);
    out.block = block;
    out.records = reinterpret_cast<uint32_t*>(bp);
    out.attrs = reinterpret_cast<uint32_t*>(bp + rec_b);
    out.cwords = compact ? reinterpret_cast<uint32_t*>(bp + rec_b + attr_b) : nullptr;
    out.words = reinterpret_cast<uint2*>(bp + rec_b + attr_b + cw_b);
    out.node_count = nodes;
    out.attr_count = leaves;
    tr.mark(s, "alloc out");

    const uint32_t zero = 0;
    cudaMemcpyAsync(codes_a, &zero, sizeof(zero), cudaMemcpyHostToDevice, s);
    uint32_t first = 0;
    for (uint32_t L = 0; L < depth; ++L) {
        const uint32_t nl = static_cast<uint32_t>(N[L]);
        child_counts<<<grid_for(nl), kThreads, 0, s>>>(codes_a, nl, V[L], cnt);
        if (cudaError_t e = cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, cnt, excl, static_cast<int>(nl), s);
            e != cudaSuccess)
            return e;
        LevelArgs a{};
        a.codes = codes_a;
        a.n = nl;
        a.v = V[L];
        a.excl = excl;
        a.first = first;
        a.next_first = first + nl;
        a.last = L + 1 == depth;
        a.records = out.records;
        a.cwords = out.cwords;
        a.next_codes = codes_b;
        a.attrs = out.attrs;
        a.color_mode = color_mode;
        a.color_constant = color_constant;
        a.resolution = n;
        if (a.last)
            emit_leaves<<<grid_for(nl), kThreads, 0, s>>>(a);
        else
            emit_level<<<grid_for(nl), kThreads, 0, s>>>(a);
        first += nl;
        std::swap(codes_a, codes_b);
    }
    if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
    tr.mark(s, "levels");
    return cudaSuccess;
}

} // namespace vxa
