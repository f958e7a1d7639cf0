// voxanim-b200: GPU extensions of the drop-in API (not in the reference).
//
// render_frame() (renderer.hpp) is the reference-compatible entry point;
// render_frame_ex() exposes what the reference's signature cannot carry:
// the kernel precision, the multi-GPU screen-tile partition and per-pixel
// parity outputs (hit object, leaf parent node, attribute index, level,
// voxel, t). Both go through the C ABI in include/vxa.h.
#pragma once

#include <cstdint>
#include <vector>

#include "vxa.h"
#include "voxanim/ingest.hpp"
#include "voxanim/renderer.hpp"

namespace voxanim::gpu {

enum class Precision : std::uint8_t {
    FP32 = VXA_FP32, // production kernel
    FP64 = VXA_FP64, // parity kernel (bit-exact with the reference CPU renderer)
};

struct RenderOptionsEx {
    Precision precision = Precision::FP32;
    int tile_rank = 0;  // screen-tile partition of the frame (64x64 super-tiles,
    int tile_world = 1; // round-robin); 1 = whole frame on this device
    std::vector<vxa_pixel_aov>* aov = nullptr; // resized to width*height when set
    bool read_image = true; // false: the frame stays in HBM, the returned Image is empty
};

// Default precision of render_frame(): VOXANIM_PRECISION=fp64|fp32 (fp32 if unset).
Precision default_precision();
void set_default_precision(Precision p);

Image render_frame_ex(const Scene& scene, const RenderOptions& opts, const RenderOptionsEx& ex, FrameStats& stats,
                      vxa_stats* device_stats = nullptr);

// Same frame written straight into a caller-owned RGB8 buffer (width*height*3
// bytes, or null to keep the frame in HBM only); the API's Image is skipped.
void render_frame_into(const Scene& scene, const RenderOptions& opts, const RenderOptionsEx& ex, FrameStats& stats,
                       std::uint8_t* rgb_out, vxa_stats* device_stats = nullptr);

// Process-wide CUDA context (device from VOXANIM_DEVICE, default 0).
vxa_ctx* context();

// Device handle of a model, uploading it on first use. Scene models
// (shared_ptr<const SvoModel>, scene.hpp:20) are keyed by their owner (a
// weak_ptr holds the control block, so the key is never reused by another
// model; the device copy is released once the model is destroyed) plus a
// storage/content check; a bare reference (traverse API) is keyed by its
// storage (node/attribute buffers, sizes, depth) plus a content signature.
std::uint32_t model_handle(const std::shared_ptr<const SvoModel>& model);
std::uint32_t model_handle(const SvoModel& model);
// Starts assembling a frame's instance table: handles returned from here on are
// not evicted by the model cache until the next call.
std::uint64_t begin_model_frame();

// voxanim::build_from_grid on the device (vxa_build_model): the same SvoModel,
// byte for byte, built in HBM and copied back; the device copy is kept in the
// model cache, so rendering the returned model does not upload it again.
SvoModel build_from_grid(const VoxelGrid& grid, std::uint32_t depth);

// Translates a vxa_status into the API's exception types (throws unless VXA_OK).
void check(int status, const char* what);

} // namespace voxanim::gpu
