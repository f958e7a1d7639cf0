/*
 * vxa.h — C ABI of the voxanim-b200 CUDA layer (sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path. The reference is
 * a C++20 library whose frame entry point is
 *     voxanim::Image voxanim::render_frame(const Scene&, const RenderOptions&, FrameStats&)
 *     (proj/include/voxanim/renderer.hpp:126, proj/src/renderer.cpp:218-300)
 * and whose per-ray kernel is
 *     std::optional<TraversalHit> voxanim::traverse(const SvoModel&, const Ray&, const OctreeBounds&)
 *     (proj/include/voxanim/traversal.hpp:62-63, proj/src/traversal.cpp:249-252).
 * Host C++ (libvoxanim.so, the same voxanim:: API) calls into this ABI; a
 * maintainer of the reference who wants the GPU path links libvxa.so and
 * replaces those two functions with the calls below.
 *
 * Conventions: plain C types only; every call returns a vxa_status; on
 * failure vxa_last_error() returns a thread-local message. No exceptions
 * cross this boundary. All FP inputs are IEEE doubles exactly as held by
 * the reference types (RigidTransform, Camera, Ray); the library derives its
 * FP32 working set from them.
 */
#ifndef VXA_H
#define VXA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VXA_ABI_VERSION 1

typedef enum vxa_status {
    VXA_OK = 0,
    VXA_ERR_INVALID = 1,   /* bad argument / dimension mismatch  -> voxanim::ValidationError */
    VXA_ERR_MODEL = 2,     /* model violates the SVO invariants  -> voxanim::ValidationError */
    VXA_ERR_CUDA = 3,      /* CUDA runtime failure               -> voxanim::DeviceError */
    VXA_ERR_OOM = 4,       /* device allocation failed           -> voxanim::DeviceError */
    VXA_ERR_NO_DEVICE = 5  /* no usable sm_100 device            -> voxanim::DeviceError */
} vxa_status;

typedef enum vxa_precision {
    VXA_FP32 = 0, /* production kernel: FP32 traversal, decisions identical except slab-test ties */
    VXA_FP64 = 1  /* parity kernel: reference operation order in FP64, bit-exact vs the CPU renderer */
} vxa_precision;

typedef struct vxa_ctx vxa_ctx;

/* ---- context ------------------------------------------------------------ */

/* One context drives one CUDA device (one process per GPU; multi-GPU frames
 * use the screen-tile partition in vxa_frame_desc plus vxa_fb_export/import).
 * device < 0 selects VOXANIM_DEVICE or 0. */
int vxa_create(int device, vxa_ctx** out);
int vxa_destroy(vxa_ctx* ctx);
const char* vxa_last_error(void);
int vxa_abi_version(void);
/* Device ordinal, SM count, and the kernel build tag (for logs). */
int vxa_device_info(vxa_ctx* ctx, int* device, int* sm_count, char* name, size_t name_len);

/* ---- models ------------------------------------------------------------- */

/* Uploads one SvoModel. `nodes` is node_count records in the 12-byte
 * voxanim::SvoNode layout {u32 child_base, u32 attr_base, u8 valid, u8 leaf,
 * u16 pad} (proj/include/voxanim/svo.hpp:28-35); `attrs` is attr_count RGBA8
 * records (VoxelAttribute). The model is checked with the reference's
 * validate() rules (proj/src/svo.cpp:134-172) and repacked on the device.
 * Node indices on the device equal indices into `nodes`. */
int vxa_upload_model(vxa_ctx* ctx, const void* nodes, uint32_t node_count, const void* attrs,
                     uint32_t attr_count, uint32_t depth, uint32_t* handle_out);
int vxa_release_model(vxa_ctx* ctx, uint32_t handle);
/* Uploads a model straight from its .svo byte stream (the format of reference
 * proj/src/svo.cpp:205-229): the header is checked like deserialize()
 * (svo.cpp:231-291) and the 12-byte node records are uploaded in place (no host
 * SvoModel). On a format error returns VXA_ERR_MODEL and, if format_error is
 * non-null, stores the voxanim::SvoFormatErrorCode (errors.hpp: 0 BadMagic,
 * 1 BadVersion, 2 BadHeader, 3 Truncated, 4 TrailingData, 5 NodeIndexOutOfRange,
 * 6 AttrIndexOutOfRange); -1 when the stream is well-formed. */
int vxa_upload_svo(vxa_ctx* ctx, const uint8_t* bytes, size_t size, uint32_t* handle_out, int32_t* format_error);
/* Device-side size of a model: bytes of the packed node words and attributes,
 * and which packed format was chosen (1 = 4-byte words, 2 = 8-byte words). */
int vxa_model_info(vxa_ctx* ctx, uint32_t handle, uint64_t* device_bytes, uint32_t* node_format);

/* Device model build: replaces voxanim::build_from_grid (reference
 * proj/include/voxanim/svo.hpp:62, proj/src/svo.cpp:52-132) for a dense grid.
 * grid_words: host copy of a VoxelGrid bitset (proj/include/voxanim/ingest.hpp:34-63:
 * resolution n = 2^depth, bit (x*n + y)*n + z of 64-bit words, (n^3+63)/64 words);
 * depth in [1, 10] (the dense-grid cap, ingest.cpp:15). color_mode: the grid's
 * ColorSpec (0 PositionHash, 1 ByHeight, 2 Constant with color_rgba = r | g<<8 |
 * b<<16 | a<<24). The model is built in device memory (same node and attribute
 * numbering as the reference, byte for byte) and registered like an upload;
 * node_count / attr_count (optional) receive its size. The context keeps its
 * build scratch (grid staging, occupancy pyramid, level lists; ~1.5 GB after a
 * depth-10 build) for the next build until vxa_destroy. */
int vxa_build_model(vxa_ctx* ctx, const uint64_t* grid_words, uint32_t depth, uint32_t color_mode,
                    uint32_t color_rgba, uint32_t* handle_out, uint64_t* node_count, uint64_t* attr_count);
/* Copy a device model's 12-byte SvoNode records and attributes to host memory
 * (either pointer may be null; capacities in elements). */
int vxa_model_download(vxa_ctx* ctx, uint32_t handle, void* nodes, uint64_t node_cap, uint32_t* attrs,
                       uint64_t attr_cap);
int vxa_model_counts(vxa_ctx* ctx, uint32_t handle, uint32_t* depth, uint64_t* node_count, uint64_t* attr_count);

/* ---- frame -------------------------------------------------------------- */

/* voxanim::Camera (proj/include/voxanim/scene.hpp:35-42). */
typedef struct vxa_camera {
    double position[3];
    double orientation[9]; /* row-major; columns right, up, back */
    double vertical_fov_deg;
    int32_t width;
    int32_t height;
} vxa_camera;

/* One voxanim::SceneObject (scene.hpp:17-23): model + id + RigidTransform
 * (math.hpp:158-169) + dirty flag. */
typedef struct vxa_instance {
    uint32_t model;
    int32_t id;
    double rotation[9];
    double translation[3];
    double scale[3];
    uint8_t dirty;
    uint8_t pad[7];
} vxa_instance;

/* Per-pixel hit record in the host voxanim::HitRecord layout
 * (renderer.hpp:32-41): 48 bytes. Used for the hit buffer (HBO). */
typedef struct vxa_hit_record {
    uint8_t color[4];
    uint8_t pad0[4];
    double normal[3];
    double t;
    int32_t object_id;
    uint8_t kind; /* 0 Miss, 1 SingleSphere, 2 MultiSphere */
    uint8_t pad1[3];
} vxa_hit_record;

typedef struct vxa_frame_desc {
    vxa_camera camera;
    uint8_t background[3];
    uint8_t culling;      /* RenderOptions::culling */
    uint8_t sorting;      /* RenderOptions::sorting */
    uint8_t precision;    /* vxa_precision */
    uint8_t camera_dirty; /* Camera::dirty, read by the HBO reuse rule */
    uint8_t pad0;
    int32_t tile_rank;    /* screen-tile partition: this device renders the 64x64 */
    int32_t tile_world;   /* super-tiles s with s % tile_world == tile_rank (1 = all) */
    /* Host hit buffer (width*height records) or NULL (RenderOptions::hbo).
     * Read before and written after the frame, in place. */
    vxa_hit_record* hbo;
    /* Device-resident hit buffer (vxa_hbo_create handle) or 0: same reuse rule,
     * records stay in HBM between frames (the paper's frame-coherence buffer
     * without host round trips). Mutually exclusive with hbo. */
    uint32_t hbo_device;
    uint32_t pad1;
} vxa_frame_desc;

/* voxanim::FrameStats (renderer.hpp:62-68) plus device evidence. */
typedef struct vxa_stats {
    uint64_t rays;
    uint64_t sphere_tests;
    uint64_t svo_traversals;
    uint64_t pixels_reused;
    uint64_t node_fetches;   /* internal-node words loaded (8 B algorithmic each) */
    uint64_t leaf_hits;      /* attribute fetches (4 B each) */
    uint64_t kernel_launches;/* kernels this call launched */
    double gpu_ms;           /* CUDA-event time of the frame kernels on the context stream */
    uint64_t h2d_bytes;      /* host->device bytes the call(s) copied (instance table, hit buffer) */
    uint64_t d2h_bytes;      /* device->host bytes (image, AOVs, hit buffer, counters) */
    uint64_t frames;         /* frames submitted (gpu_ms covers them; kernel_launches also counts pre-passes) */
} vxa_stats;

/* Per-pixel parity outputs (host array of width*height, row-major). */
typedef struct vxa_pixel_aov {
    double t;             /* hit parameter (world == local, rotations preserve length) */
    int32_t object_id;    /* -1: miss */
    uint32_t node_index;  /* parent node of the hit leaf (index into SvoModel::nodes) */
    uint32_t attr_index;  /* index into SvoModel::attributes */
    uint32_t voxel[3];    /* leaf_path_to_voxel of the hit path */
    uint8_t level;        /* path_len */
    uint8_t kind;         /* HitKind */
    uint8_t entry_axis;   /* axis of the entry face (normal_local axis), 0..2 */
    uint8_t pad0;
    uint32_t traversals;  /* SVO traversals started for this pixel */
    uint32_t node_fetches;/* internal-node words loaded for this pixel */
    uint32_t pad1;
} vxa_pixel_aov;

/* Renders one frame synchronously. instances are in scene order. rgb_out:
 * host RGB8 (width*height*3) or NULL to keep the frame on the device only.
 * aov_out: host array or NULL. stats may be NULL. */
int vxa_render(vxa_ctx* ctx, const vxa_frame_desc* frame, const vxa_instance* instances,
               uint32_t instance_count, uint8_t* rgb_out, vxa_pixel_aov* aov_out, vxa_stats* stats);

/* Device-resident hit buffers (HBO) for width x height frames, initialised
 * to Miss records (a fresh voxanim::HitBuffer). */
int vxa_hbo_create(vxa_ctx* ctx, int32_t width, int32_t height, uint32_t* handle_out);
int vxa_hbo_release(vxa_ctx* ctx, uint32_t handle);
/* Copies a device hit buffer to host records (width*height), and back. */
int vxa_hbo_download(vxa_ctx* ctx, uint32_t handle, vxa_hit_record* out);
int vxa_hbo_upload(vxa_ctx* ctx, uint32_t handle, const vxa_hit_record* in);

/* Asynchronous form for benchmarking: enqueues the frame on the context
 * stream (framebuffer stays in HBM), no host outputs; a device hit buffer
 * (hbo_device) is allowed, a host one is not. */
int vxa_submit(vxa_ctx* ctx, const vxa_frame_desc* frame, const vxa_instance* instances,
               uint32_t instance_count);
int vxa_synchronize(vxa_ctx* ctx);

/* Streaming form: enqueues the frame, its RGB8 pack and an asynchronous D2H into
 * rgb_out (host, width*height*3; page-lock it with vxa_host_register) on a copy
 * stream, so frame k's readback overlaps frame k+1's kernel. Returns a ticket;
 * rgb_out is valid once vxa_wait_readback(ticket) returns. Two readbacks can be
 * in flight; a third waits for the oldest. */
int vxa_submit_readback(vxa_ctx* ctx, const vxa_frame_desc* frame, const vxa_instance* instances,
                        uint32_t instance_count, uint8_t* rgb_out, uint64_t* ticket);
int vxa_wait_readback(vxa_ctx* ctx, uint64_t ticket);
/* Device counters accumulated since the last vxa_stats_reset. */
int vxa_stats_read(vxa_ctx* ctx, vxa_stats* stats);
int vxa_stats_reset(vxa_ctx* ctx);
/* Copies the resident RGBA8 framebuffer to host RGB8 (width*height*3). */
int vxa_read_framebuffer(vxa_ctx* ctx, uint8_t* rgb_out, int32_t width, int32_t height);

/* Page-locks a caller-owned host buffer (cudaHostRegister) so image / AOV
 * reads into it run as asynchronous DMA at full PCIe rate; unregister before
 * freeing the memory. */
int vxa_host_register(vxa_ctx* ctx, void* ptr, size_t bytes);
int vxa_host_unregister(vxa_ctx* ctx, void* ptr);

/* Timing helpers on the context stream (CUDA events). */
int vxa_timer_begin(vxa_ctx* ctx);
int vxa_timer_end(vxa_ctx* ctx, double* elapsed_ms);
/* Writes a scratch buffer larger than L2 on the context stream. */
int vxa_flush_l2(vxa_ctx* ctx);
/* Holds the context stream for about `microseconds` (one spinning thread):
 * enqueued before vxa_timer_begin it gives the host time to enqueue the timed
 * work, so host submission latency stays out of a device-timed region. */
int vxa_stream_delay(vxa_ctx* ctx, uint32_t microseconds);
/* Raw cudaStream_t of the context (for callers that record their own events). */
void* vxa_stream(vxa_ctx* ctx);

/* ---- multi-GPU framebuffer gather over NVLink --------------------------- */

/* Rank 0 exports its framebuffer (allocated for width x height) as a CUDA IPC
 * handle (64 bytes); every other rank imports it, after which its frames
 * store their super-tiles straight into rank 0's framebuffer through the
 * peer mapping (NVLink / NVSwitch). */
int vxa_fb_export(vxa_ctx* ctx, int32_t width, int32_t height, void* ipc_handle_out);
int vxa_fb_import(vxa_ctx* ctx, int32_t width, int32_t height, const void* ipc_handle); /* NULL: detach */

/* Frame completion across ranks without a host barrier. The reference's frame
 * is complete when every row-band thread has joined (renderer.cpp:268-287);
 * across GPUs the same point is "every rank's super-tiles are in rank 0's
 * framebuffer". Rank 0 exports a small flag block {go, done[world]} in its HBM
 * (vxa_sync_export, 64-byte CUDA IPC handle); every other rank imports it.
 * Per frame, every rank calls vxa_frame_open before submitting and
 * vxa_frame_close after it (the same number of times on every rank; frames are
 * numbered by the calls):
 *   rank 0: open stores go = frame; close waits until done[r] == frame for all r;
 *   rank r: open waits until go == frame; close stores done[r] = frame.
 * mode VXA_SYNC_DEVICE: the stores and waits are 1-thread kernels on the
 * context stream (system-scope release stores / acquire loads over NVLink),
 * so the host never blocks and rank 0's stream ends the frame only when the
 * whole frame has landed; a wait gives up after timeout_ms and latches an
 * error that vxa_sync_status reports. Only for ranks on distinct GPUs: kernels
 * that wait on one another must never share a device.
 * mode VXA_SYNC_HOST: the waits are host polls of the flags (ranks sharing one
 * device: a correctness run of the same protocol). */
#define VXA_SYNC_DEVICE 0
#define VXA_SYNC_HOST 1
int vxa_sync_export(vxa_ctx* ctx, int32_t world, void* ipc_handle_out);
int vxa_sync_import(vxa_ctx* ctx, int32_t rank, int32_t world, const void* ipc_handle);
int vxa_sync_configure(vxa_ctx* ctx, int32_t mode, uint32_t timeout_ms);
int vxa_frame_open(vxa_ctx* ctx);
int vxa_frame_close(vxa_ctx* ctx);
/* 0 when no wait has timed out (synchronises the context stream). */
int vxa_sync_status(vxa_ctx* ctx, int32_t* timed_out);
/* Streaming readback of the resident (composed) framebuffer: its RGB8 pack on
 * the context stream (after everything enqueued so far, e.g. vxa_frame_close)
 * and the D2H into rgb_out on the copy stream; same tickets as
 * vxa_submit_readback. */
int vxa_framebuffer_readback(vxa_ctx* ctx, int32_t width, int32_t height, uint8_t* rgb_out, uint64_t* ticket);

/* Screen partition used when tile_world > 1: the rank that renders pixel
 * (x, y) of a width-wide frame split over `world` devices (64x64 super-tiles,
 * round-robin). Pure function, no device needed. */
int32_t vxa_tile_owner(int32_t x, int32_t y, int32_t width, int32_t height, int32_t world);

/* Composition without CUDA IPC (a collective gather instead of peer stores):
 * rank `rank`'s super-tiles (s % world == rank, ascending s) as a tile-major
 * device buffer of 64x64 RGBA8 pixels per tile (edge tiles padded).
 * vxa_tiles_count: tiles of that rank (pure function); vxa_tiles_pack copies
 * them out of this context's framebuffer into `dst` (device memory);
 * vxa_tiles_unpack writes another rank's packed tiles into this context's
 * framebuffer (rank 0 composing the frame). Both are ordered on the context
 * stream (vxa_synchronize before handing `dst` to another stream). */
int vxa_tiles_count(int32_t width, int32_t height, int32_t rank, int32_t world, uint32_t* count);
int vxa_tiles_pack(vxa_ctx* ctx, int32_t width, int32_t height, int32_t rank, int32_t world, void* dst_device);
int vxa_tiles_unpack(vxa_ctx* ctx, int32_t width, int32_t height, int32_t rank, int32_t world, const void* src_device);

/* ---- single-ray traversal (voxanim::traverse / traverse_debug) ---------- */

typedef struct vxa_local_ray {
    double origin[3];
    double direction[3];
    double half_extent[3]; /* OctreeBounds::half_extent */
} vxa_local_ray;

typedef struct vxa_traverse_hit {
    double t_hit, t_enter, t_exit;
    double normal_local[3];
    uint8_t attribute[4];
    uint32_t attr_index;
    uint32_t node_index;  /* parent node of the hit leaf */
    uint8_t leaf_path[16];
    uint8_t path_len;
    uint8_t hit;          /* 0: std::nullopt */
    uint16_t pad;
    uint32_t node_fetches;
    uint32_t log_count;   /* visits recorded (<= capacity) */
    uint32_t log_total;   /* visits that occurred */
} vxa_traverse_hit;

typedef struct vxa_visit {
    double t_enter;
    uint8_t level;
    uint8_t leaf;
    uint8_t pad[6];
} vxa_visit;

/* Batched traversal of local rays against one model. log may be NULL;
 * otherwise ray i writes up to log_capacity visits at log[i*log_capacity]. */
int vxa_traverse(vxa_ctx* ctx, uint32_t model, const vxa_local_ray* rays, uint32_t ray_count,
                 uint32_t precision, vxa_traverse_hit* hits, vxa_visit* log, uint32_t log_capacity);

#ifdef __cplusplus
}
#endif

#endif /* VXA_H */
