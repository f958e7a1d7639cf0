// Internal declarations shared by the C ABI (vxa_abi.cu) and the kernel
// translation units (render_fp32.cu: production FP32 instantiation;
// render_fp64.cu: FP64 parity instantiation, compiled with -fmad=false).
#pragma once

#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

#include "vxa_device.cuh"

namespace vxa {

// Zero-direction path bits of one axis (host + device, identical FP64 ops):
// the reference tracks the node centre along an axis the ray never moves on
// (centre_{L+1} = centre_L +/- ldexp(h, -(L+1)), traversal.cpp:135-170) and
// takes the upper child iff !(centre > o). Only the child containing o can
// have a non-empty interval, so the whole descent is this one bit sequence.
__host__ __device__ inline uint32_t zero_dir_bits(double o, double h) {
    uint32_t bits = 0;
    double c = 0.0;
    for (int L = 0; L < static_cast<int>(kMaxDepth); ++L) {
        const bool upper = !(c > o);
        if (upper) bits |= 1u << L;
        const double q = ldexp(h, -(L + 1));
        c = upper ? c + q : c - q;
    }
    return bits;
}

struct FrameLaunch {
    int grid;
    cudaStream_t stream;
};

// Node words the FP32 frame kernel stages in shared memory (0 = off; build variant).
constexpr uint32_t kSmemTopWords = VXA_SMEM_TOP;
// Per-super-tile candidate lists for large scenes (frame_kernel.cuh: super_cull_kernel).
cudaError_t launch_super_cull(const FrameParams<float>& p, uint16_t* list, uint32_t* count, uint32_t* done,
                              cudaStream_t s);
cudaError_t launch_super_cull(const FrameParams<double>& p, uint16_t* list, uint32_t* count, uint32_t* done,
                              cudaStream_t s);
cudaError_t launch_frame_f32(const FrameParams<float>& p, bool aov, bool hbo, const FrameLaunch& l);
cudaError_t launch_frame_f64(const FrameParams<double>& p, bool aov, bool hbo, const FrameLaunch& l);
// hbo: 0 none, 1 48-byte records, 2 16-byte records (FP32 only)
int frame_blocks_per_sm_f32(bool aov, int hbo, bool compact, uint32_t max_depth);
int frame_blocks_per_sm_f64(bool aov, int hbo, bool compact, uint32_t max_depth);
size_t frame_smem_bytes_f32(uint32_t max_depth);

size_t frame_smem_bytes_f64(uint32_t max_depth);

struct TraverseRayIn {
    double origin[3];
    double direction[3];
    double half_extent[3];
};

struct TraverseRayOut {
    double t_hit, t_enter, t_exit;
    double normal_local[3];
    uint8_t attribute[4];
    uint32_t attr_index;
    uint32_t node_index;
    uint8_t leaf_path[16];
    uint8_t path_len;
    uint8_t hit;
    uint16_t pad;
    uint32_t node_fetches;
    uint32_t log_count;
    uint32_t log_total;
};

struct VisitOut {
    double t_enter;
    uint8_t level;
    uint8_t leaf;
    uint8_t pad[6];
};

cudaError_t launch_traverse_f64(const DevModel& m, const TraverseRayIn* rays, uint32_t n, TraverseRayOut* out,
                                VisitOut* log, uint32_t log_cap, cudaStream_t s);
cudaError_t launch_traverse_f32(const DevModel& m, const TraverseRayIn* rays, uint32_t n, TraverseRayOut* out,
                                VisitOut* log, uint32_t log_cap, cudaStream_t s);

// Grow-only device scratch kept by a context between calls.
struct Arena {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        cudaFree(p);
        p = nullptr;
        cap = 0;
        const cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// Device build of a dense grid (build.cu; reference svo.cpp:52-132).
struct BuildScratch {
    Arena grid, pyramid, levels;
};
struct BuiltModel {
    void* block = nullptr;       // one allocation holding everything below
    uint32_t* records = nullptr; // 12-byte SvoNode records
    uint32_t* attrs = nullptr;
    uint32_t* cwords = nullptr;  // compact render words (null when bases exceed 24 bits)
    uint2* words = nullptr;      // wide render words (filled by the caller's repack)
    uint64_t node_count = 0, attr_count = 0;
    // device scalar (in the builder's scratch): float bits of the squared leaf
    // extent about the cube centre (unit-cube coordinates); valid once s is done
    const unsigned int* extent_dev = nullptr;
};
// Enqueues the build on s (returns after the level sizes are known; the
// emission passes are still in flight). On error out.block may be set.
cudaError_t build_svo(cudaStream_t s, const uint64_t* grid_dev, uint32_t depth, uint32_t color_mode,
                      uint32_t color_constant, BuildScratch& scratch, BuiltModel& out);

} // namespace vxa
