// C ABI of the CUDA layer (include/vxa.h): device context, model cache and
// repack, per-frame instance constants, frame submission, readback, timing
// and the multi-GPU framebuffer mapping.
//
// Host arithmetic in this file feeds the FP64 parity kernel, so it is written
// in the reference's operand order (bounding_sphere scene.cpp:16-20,
// transform_ray_world_to_local math.hpp:206-224, bounds_from_scale
// traversal.hpp:21-23, ray_box_params traversal.cpp:30-61) and compiled with
// -ffp-contract=off.
#include "vxa.h"

#include <cuda.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "vxa_internal.h"

using namespace vxa;

namespace {

thread_local std::string g_error;

int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

#define VXA_CUDA(call)                                                                                    \
    do {                                                                                                  \
        const cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                            \
            return fail(e_ == cudaErrorMemoryAllocation ? VXA_ERR_OOM : VXA_ERR_CUDA,                     \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                              \
    } while (0)

// ---------------------------------------------------------------------------
// device helper kernels

// 12-byte SvoNode records -> packed {valid | leaf << 8 | mixed, base} words.
__global__ void repack_nodes(const uint32_t* __restrict__ raw, uint32_t n, uint2* __restrict__ words,
                             uint32_t* __restrict__ side) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t child_base = raw[3 * i], attr_base = raw[3 * i + 1], masks = raw[3 * i + 2];
    const uint32_t valid = masks & 0xffu, leaf = (masks >> 8) & 0xffu;
    const uint32_t internal = valid & ~leaf & 0xffu, leaves = valid & leaf;
    uint2 w;
    w.x = valid | (leaf << 8) | ((internal && leaves) ? kMixed : 0u);
    w.y = internal ? child_base : attr_base;
    words[i] = w;
    // child_base is unique among nodes with internal children
    if (side != nullptr && internal && leaves) side[child_base] = attr_base;
}

// Fresh hit records: HitRecord{} (colour {0,0,0,255}, normal 0, t 0, id -1, Miss).
__global__ void init_hit_records(HitRec* r, size_t n) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    HitRec h;
    h.color = 0xff000000u;
    h.pad0 = 0;
    h.normal[0] = h.normal[1] = h.normal[2] = 0.0;
    h.t = 0.0;
    h.object_id = -1;
    h.kind = 0;
    h.pad1[0] = h.pad1[1] = h.pad1[2] = 0;
    r[i] = h;
}

// RGBA8 framebuffer -> RGB8 (four pixels per thread: 16 B in, 12 B out).
__global__ void pack_rgb(const uint32_t* __restrict__ fb, uint8_t* __restrict__ rgb, size_t n_pix) {
    const size_t q = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t p0 = q * 4;
    if (p0 >= n_pix) return;
    if (p0 + 4 <= n_pix) {
        const uint4 v = reinterpret_cast<const uint4*>(fb)[q];
        const uint32_t a = (v.x & 0xffffffu) | (v.y << 24);
        const uint32_t b = ((v.y >> 8) & 0xffffu) | (v.z << 16);
        const uint32_t c = ((v.z >> 16) & 0xffu) | (v.w << 8);
        uint32_t* dst = reinterpret_cast<uint32_t*>(rgb + p0 * 3);
        dst[0] = a;
        dst[1] = b;
        dst[2] = c;
    } else {
        for (size_t p = p0; p < n_pix; ++p) {
            const uint32_t v = fb[p];
            rgb[3 * p] = static_cast<uint8_t>(v);
            rgb[3 * p + 1] = static_cast<uint8_t>(v >> 8);
            rgb[3 * p + 2] = static_cast<uint8_t>(v >> 16);
        }
    }
}

// ---- compact device hit buffers (FP32 frames) --------------------------------
// Local normal (axis, sign) of a world normal n of an object with rotation R:
// n_local = R^T n, the axis of largest magnitude.
__device__ __forceinline__ uint32_t local_normal_meta(const float* R, const double n[3]) {
    float best = -1.0f;
    uint32_t axis = 0, neg = 0;
    for (uint32_t a = 0; a < 3; ++a) {
        const float v = R[a] * static_cast<float>(n[0]) + R[3 + a] * static_cast<float>(n[1]) +
                        R[6 + a] * static_cast<float>(n[2]);
        if (fabsf(v) > best) best = fabsf(v), axis = a, neg = v < 0.0f ? 1u : 0u;
    }
    return (axis << 2) | (neg << 4);
}

// Instance of an object id: binary search of a (id, first instance index) table
// sorted by id (the reference's find_object rule: the first object with the id).
__device__ __forceinline__ int find_instance(const int2* __restrict__ map, uint32_t n, int32_t id) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (map[mid].x < id) lo = mid + 1;
        else hi = mid;
    }
    return (lo < n && map[lo].x == id) ? map[lo].y : -1;
}

// 48-byte records -> 16-byte ones against the frame's instance table.
__global__ void hbo_compress(const HitRec* __restrict__ in, HitRec16* __restrict__ out, size_t n,
                             const DevInstance<float>* __restrict__ inst, const int2* __restrict__ map,
                             uint32_t map_n) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const HitRec r = in[i];
    HitRec16 c;
    c.color = r.color;
    c.t = static_cast<float>(r.t);
    c.object_id = r.object_id;
    c.meta = r.kind & 3u;
    if (r.kind != 0) {
        const int k = find_instance(map, map_n, r.object_id);
        if (k >= 0) c.meta |= local_normal_meta(inst[k].R, r.normal);
    }
    out[i] = c;
}

// The rotation of every instance of an FP32 frame (for later expansion).
__global__ void hbo_save_table(const DevInstance<float>* __restrict__ inst, uint32_t n_inst, float* __restrict__ tab) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_inst) return;
    for (int j = 0; j < 9; ++j) tab[9 * k + j] = inst[k].R[j];
}

// 16-byte records -> 48-byte host-layout ones: the normal is +-column `axis` of
// the object's R (the FP32 kernel's best_normal), as the 48-byte path stores it.
__global__ void hbo_expand(const HitRec16* __restrict__ in, HitRec* __restrict__ out, size_t n,
                           const float* __restrict__ tab, const int2* __restrict__ map, uint32_t map_n) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const HitRec16 c = in[i];
    HitRec r;
    r.color = c.color;
    r.pad0 = 0;
    r.normal[0] = r.normal[1] = r.normal[2] = 0.0;
    r.t = static_cast<double>(c.t);
    r.object_id = c.object_id;
    r.kind = static_cast<uint8_t>(c.meta & 3u);
    r.pad1[0] = r.pad1[1] = r.pad1[2] = 0;
    if (r.kind != 0) {
        const uint32_t axis = (c.meta >> 2) & 3u;
        const bool neg = (c.meta & 16u) != 0;
        const int k = find_instance(map, map_n, c.object_id);
        if (k >= 0)
            for (int j = 0; j < 3; ++j) {
                const float v = tab[9 * k + 3 * j + axis];
                r.normal[j] = static_cast<double>(neg ? -v : v);
            }
    }
    out[i] = r;
}

struct ModelEntry {
    DevModel dev{};
    uint2* words = nullptr;
    uint32_t* cwords = nullptr; // compact words when the model is canonical
    uint32_t* side = nullptr;
    uint32_t* attrs = nullptr;
    uint32_t* raw = nullptr; // the 12-byte SvoNode records (vxa_model_download)
    void* block = nullptr;   // device-built models: one allocation holds all of the above
    uint64_t attr_count = 0;
    uint64_t bytes = 0;
    void free_all() {
        if (block) {
            cudaFree(block);
        } else {
            cudaFree(words);
            cudaFree(cwords);
            cudaFree(side);
            cudaFree(attrs);
            cudaFree(raw);
        }
        block = nullptr;
        words = nullptr;
        cwords = nullptr;
        side = nullptr;
        attrs = nullptr;
        raw = nullptr;
    }
};

template <typename T> struct DevBuf {
    T* ptr = nullptr;
    size_t cap = 0; // elements
    cudaError_t ensure(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        const cudaError_t e = cudaMalloc(&ptr, std::max<size_t>(n, 1) * sizeof(T));
        if (e == cudaSuccess) cap = n;
        return e;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

} // namespace

struct vxa_ctx {
    // Serialises the API calls on this context (its buffers, streams and
    // counters are shared state); recursive: some entry points call others.
    std::recursive_mutex mu;
    int device = 0;
    int sm_count = 0;
    char name[256] = {};
    cudaStream_t stream = nullptr;
    std::map<uint32_t, ModelEntry> models;
    uint32_t next_handle = 1;
    BuildScratch build; // vxa_build_model scratch (grid staging, pyramid, level lists)

    DevBuf<uint32_t> fb;  // resident RGBA8 framebuffer
    int32_t fb_w = 0, fb_h = 0;
    uint32_t* peer_fb = nullptr; // rank 0's framebuffer mapped via CUDA IPC
    int32_t peer_w = 0, peer_h = 0;

    // Frame completion flags (vxa_frame_open/close): rank 0 owns the block
    // {go, pad, done[kSyncRanks]} in its HBM, other ranks map it via CUDA IPC.
    static constexpr int kSyncRanks = 64;
    DevBuf<unsigned int> sync_own;     // rank 0: the flag block
    unsigned int* sync_peer = nullptr; // rank r: rank 0's block, peer-mapped
    unsigned int* sync_flags = nullptr; // the block this rank addresses (own or peer)
    DevBuf<unsigned int> sync_err;     // latched by a wait that timed out
    int32_t sync_rank = 0, sync_world = 1;
    int32_t sync_mode = VXA_SYNC_DEVICE;
    uint64_t sync_timeout_ns = 10ull * 1000 * 1000 * 1000;
    uint32_t sync_seq = 0; // frames opened so far
    cudaStream_t poll_stream = nullptr; // VXA_SYNC_HOST flag reads
    unsigned int* sync_host = nullptr;  // pinned, kSyncRanks + 2 words

    DevBuf<uint32_t> tile_counter;
    DevBuf<unsigned long long> counters;
    unsigned long long* counters_host = nullptr; // pinned, 8 counters
    // Per-frame instance tables, double-buffered on the device: frame k+1's
    // table is uploaded on upload_stream while frame k renders (the frame waits
    // for inst_done, the upload for inst_free: the kernel two frames back).
    DevBuf<unsigned char> inst_dev[2];
    cudaStream_t upload_stream = nullptr;
    cudaEvent_t inst_free[2] = {nullptr, nullptr};
    DevBuf<uint16_t> super_list;  // per-super-tile candidate lists (large scenes)
    DevBuf<uint32_t> super_count;
    DevBuf<uint32_t> super_order; // longest-first super-tile order (VXA_LPT)
    DevBuf<uint32_t> super_done;  // pre-pass block tickets (the last block sorts; reset by it)
    DevBuf<unsigned long long> tile_mask; // per-tile candidate masks over the super-tile lists
    DevBuf<int2> id_map;                  // (object id, first instance) sorted by id: hit-buffer conversions
    int aux_launches = 0;         // pre-pass kernels since the last stats reset
    unsigned char* inst_host[2] = {nullptr, nullptr};
    size_t inst_host_cap = 0;
    cudaEvent_t inst_done[2] = {nullptr, nullptr};
    int inst_slot = 0;

    struct DeviceHbo {
        HitRec* rec = nullptr;     // 48-byte host-layout records (FP64 frames, host access)
        HitRec16* rec16 = nullptr; // 16-byte records of FP32 frames (allocated on first FP32 use)
        bool compact = false;      // rec16 holds the current records
        DevBuf<float> tab;         // R (9 floats) per instance of the last FP32 frame (expansion)
        std::vector<int32_t> tab_ids; // that frame's object ids, in instance order
        uint32_t tab_n = 0;
        int32_t w = 0, h = 0;
    };
    std::map<uint32_t, DeviceHbo> hbos;
    uint32_t next_hbo = 1;
    DevBuf<PixelAov> aov;
    DevBuf<HitRec> hbo;
    DevBuf<uint8_t> rgb;
    DevBuf<unsigned char> l2_scratch;
    DevBuf<TraverseRayIn> rays;
    DevBuf<TraverseRayOut> hits;
    DevBuf<VisitOut> visits;

    cudaEvent_t ev_a = nullptr, ev_b = nullptr, t_a = nullptr, t_b = nullptr;
    // streaming readback: RGB8 staging ring on a copy stream
    cudaStream_t copy_stream = nullptr;
    DevBuf<uint8_t> rb_rgb[2];
    cudaEvent_t rb_packed[2] = {nullptr, nullptr}, rb_done[2] = {nullptr, nullptr};
    uint64_t rb_next = 0; // next ticket
    // The newest frame's D2H is enqueued at the next submission, after that
    // frame's instance upload, so the small H2D never queues behind a 25 MB D2H
    // on a shared copy engine (the next kernel would wait for it).
    bool rb_pending = false;
    uint8_t* next_rgb = nullptr;          // RGB8 target of the frame being submitted (streaming)
    // synchronous readback in bands (vxa_render): per-band tile counters the copy
    // stream waits on (cuStreamWaitValue32), set for the frame being submitted
    DevBuf<uint32_t> band_done;
    uint32_t* next_band_done = nullptr;
    uint32_t next_band_rows = 0;
    cudaEvent_t band_reset = nullptr;
    cudaEvent_t band_trace[16] = {}; // VOXANIM_BAND_TRACE: per-band copy completion events
    cudaStream_t copy_stream2 = nullptr; // second D2H stream of the banded readback (bands alternate)
    int band_api = 0; // 0 unknown, 1 cuStreamWaitValue32 usable, -1 not
    // direct synchronous readback (vxa_render into page-locked host memory): per
    // super-tile tile counters and the device alias of the caller's image
    DevBuf<uint32_t> direct_done;
    uint32_t* next_super_done = nullptr;
    uint8_t* next_rgb_host = nullptr;
    bool next_screen_order = false; // the frame being submitted keeps the screen order of its super-tiles
    void* wait_value32 = nullptr;
    cudaEvent_t next_rgb_free = nullptr;  // its slot's previous D2H
    int rb_pending_slot = 0;
    uint8_t* rb_pending_out = nullptr;
    size_t rb_pending_bytes = 0;
    int occ[2][2][3][2][kMaxDepth + 1] = {}; // [precision][aov][hbo mode][compact][stack height]

    // Frame-kernel timing ring: events recorded tight around every frame
    // kernel launch; vxa_stats_read sums them (gpu_ms) since the last reset.
    static constexpr int kRing = 4096;
    cudaEvent_t k_begin[kRing] = {}, k_end[kRing] = {};
    int k_count = 0;
    uint64_t h2d = 0, d2h = 0; // bytes copied since the last reset
    uint64_t n_rays = 0, n_sphere_tests = 0; // host-counted (pixels rendered x objects tested)
};

namespace {

// ---------------------------------------------------------------------------
// per-frame instance constants

template <typename Real> struct HostFrame {
    std::vector<DevInstance<Real>> inst;
};

// One device instance record: everything the kernels need, folded on the host
// in FP64 in the reference's operand order and rounded once.
template <typename Real>
void fold_instance(const std::map<uint32_t, ModelEntry>& models, const vxa_frame_desc* f, const vxa_instance& s,
                   DevInstance<Real>& d) {
    const double* o = f->camera.position;
    const double* C = f->camera.orientation;
    std::memset(&d, 0, sizeof(d));
    d.id = s.id;
    d.dirty = s.dirty;
    const auto it = models.find(s.model);
    if (it == models.end()) {
        d.valid_model = 0; // reference: objects without a model are skipped (renderer.cpp:74-76)
    } else {
        d.valid_model = 1;
        d.model = it->second.dev;
    }
    const double* R = s.rotation;
    const double* t = s.translation;
    // bounding sphere: centre = translation, r = 0.5 |scale|
    const double l[3] = {t[0] - o[0], t[1] - o[1], t[2] - o[2]};
    const double L2 = l[0] * l[0] + l[1] * l[1] + l[2] * l[2];
    const double r = 0.5 * std::sqrt(s.scale[0] * s.scale[0] + s.scale[1] * s.scale[1] + s.scale[2] * s.scale[2]);
    const double r2 = r * r;
    // local ray origin: R^T (o + (-t))
    const double v[3] = {o[0] + -t[0], o[1] + -t[1], o[2] + -t[2]};
    double Rt[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Rt[3 * i + j] = R[3 * j + i];
    double ol[3];
    for (int i = 0; i < 3; ++i) ol[i] = Rt[3 * i] * v[0] + Rt[3 * i + 1] * v[1] + Rt[3 * i + 2] * v[2];
    const double h[3] = {s.scale[0] * 0.5, s.scale[1] * 0.5, s.scale[2] * 0.5};
    for (int a = 0; a < 3; ++a) {
        d.L[a] = static_cast<Real>(l[a]);
        d.A_lo[a] = static_cast<Real>(-h[a] - ol[a]);
        d.A_hi[a] = static_cast<Real>(h[a] - ol[a]);
        d.h2[a] = static_cast<Real>(2.0 * h[a]);
        d.ih2[a] = 1.0 / (2.0 * h[a]);
        // FP32 kernel: unit-cube plane offsets (-h - o) / 2h, (h - o) / 2h + residuals
        const double ulo = (-h[a] - ol[a]) / (2.0 * h[a]), uhi = (h[a] - ol[a]) / (2.0 * h[a]);
        d.U_lo[a] = static_cast<float>(ulo);
        d.U_hi[a] = static_cast<float>(uhi);
        d.Ur_lo[a] = static_cast<float>(ulo - static_cast<double>(d.U_lo[a]));
        d.Ur_hi[a] = static_cast<float>(uhi - static_cast<double>(d.U_hi[a]));
        d.zbits[a] = zero_dir_bits(ol[a], h[a]);
        if (-h[a] > ol[a]) d.zflags |= 1u << a;
        if (h[a] > ol[a]) d.zflags |= 1u << (3 + a);
    }
    d.L2 = static_cast<Real>(L2);
    d.r = static_cast<Real>(r);
    d.r2 = static_cast<Real>(r2);
    for (int i = 0; i < 9; ++i) d.R[i] = static_cast<Real>(R[i]);
    // camera -> local rotation R^T C in FP64 (FP32 kernel's local direction)
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
            for (int k2 = 0; k2 < 3; ++k2) acc += Rt[3 * i + k2] * C[3 * k2 + j];
            d.Md[3 * i + j] = acc;
        }
    if constexpr (sizeof(Real) == 8) {
        for (int i = 0; i < 9; ++i) d.M[i] = Rt[i];
    } else {
        for (int i = 0; i < 9; ++i) d.M[i] = static_cast<float>(d.Md[i]);
        // A box with a non-positive (or non-finite) extent holds no hit for the
        // reference (empty or inverted slab: the root test fails); the FP32
        // unit-cube planes would divide by 2h, so the traversal is skipped.
        for (int a = 0; a < 3; ++a)
            if (!(h[a] > 0.0) || !std::isfinite(h[a])) d.valid_model = 0;
    }
}

// Builds the device instance table in id order (index order == the
// reference's id tie-break order) straight into `out` (the pinned staging
// slot), plus the FP32 cull table; large scenes fold on several threads.
template <typename Real>
void build_instances(vxa_ctx* ctx, const vxa_frame_desc* f, const vxa_instance* in, uint32_t n, DevInstance<Real>* out,
                     float4* cull) {
    const auto by_id = [&](uint32_t a, uint32_t b) { return in[a].id < in[b].id; };
    std::vector<uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0u);
    if (!std::is_sorted(order.begin(), order.end(), by_id)) std::stable_sort(order.begin(), order.end(), by_id);
    const auto work = [&](uint32_t k0, uint32_t k1) {
        for (uint32_t k = k0; k < k1; ++k) {
            fold_instance(ctx->models, f, in[order[k]], out[k]);
            if (cull)
                cull[k] = make_float4(static_cast<float>(out[k].L[0]), static_cast<float>(out[k].L[1]),
                                      static_cast<float>(out[k].L[2]), static_cast<float>(out[k].r));
        }
    };
    const uint32_t threads = n >= 2048 ? std::min<uint32_t>(8, std::max(1u, std::thread::hardware_concurrency())) : 1;
    if (threads <= 1) {
        work(0, n);
        return;
    }
    std::vector<std::thread> pool;
    const uint32_t chunk = (n + threads - 1) / threads;
    for (uint32_t t = 1; t < threads; ++t)
        pool.emplace_back(work, std::min(n, t * chunk), std::min(n, (t + 1) * chunk));
    work(0, std::min(n, chunk));
    for (auto& th : pool) th.join();
}

template <typename Real> void fill_camera(FrameParams<Real>& p, const vxa_frame_desc* f) {
    const vxa_camera& c = f->camera;
    // std::tan on the host: the CUDA tan differs from glibc in the last ulp.
    const double tan_half = std::tan(c.vertical_fov_deg * 3.14159265358979323846 / 360.0);
    const double aspect = static_cast<double>(c.width) / c.height;
    for (int k = 0; k < 3; ++k) p.cam_pos[k] = static_cast<Real>(c.position[k]);
    for (int k = 0; k < 9; ++k) p.C[k] = static_cast<Real>(c.orientation[k]);
    p.tan_half = static_cast<Real>(tan_half);
    p.aspect = static_cast<Real>(aspect);
    p.inv_w2 = static_cast<Real>(2.0 / c.width);
    p.inv_h2 = static_cast<Real>(2.0 / c.height);
    p.sx = static_cast<Real>(tan_half * aspect);
    p.sy = static_cast<Real>(tan_half);
    p.d_kx = tan_half * aspect / c.width;
    p.d_ky = tan_half / c.height;
    p.width = c.width;
    p.height = c.height;
}

int ensure_staging(vxa_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->inst_host_cap) return VXA_OK;
    for (int s = 0; s < 2; ++s) {
        if (ctx->inst_host[s]) {
            cudaEventSynchronize(ctx->inst_done[s]);
            cudaFreeHost(ctx->inst_host[s]);
            ctx->inst_host[s] = nullptr;
        }
    }
    const size_t cap = std::max<size_t>(bytes, 64 * 1024);
    for (int s = 0; s < 2; ++s) VXA_CUDA(cudaHostAlloc(&ctx->inst_host[s], cap, cudaHostAllocDefault));
    ctx->inst_host_cap = cap;
    return VXA_OK;
}

int check_frame(const vxa_frame_desc* f) {
    if (f == nullptr) return fail(VXA_ERR_INVALID, "null frame descriptor");
    if (f->camera.width < 1 || f->camera.height < 1) return fail(VXA_ERR_INVALID, "camera resolution must be at least 1x1");
    if (f->tile_world < 1 || f->tile_rank < 0 || f->tile_rank >= f->tile_world)
        return fail(VXA_ERR_INVALID, "tile partition rank/world out of range");
    if (f->precision != VXA_FP32 && f->precision != VXA_FP64) return fail(VXA_ERR_INVALID, "unknown precision");
    return VXA_OK;
}

// Uploads the (object id, first instance index) table of `ids`, sorted by id, for
// the hit-buffer conversions; returns its length.
int upload_id_map(vxa_ctx* ctx, const int32_t* ids, uint32_t n, uint32_t* map_n) {
    std::vector<int2> m;
    m.reserve(n);
    for (uint32_t k = 0; k < n; ++k) m.push_back(make_int2(ids[k], static_cast<int>(k)));
    std::stable_sort(m.begin(), m.end(), [](const int2& a, const int2& b) { return a.x < b.x; });
    m.erase(std::unique(m.begin(), m.end(), [](const int2& a, const int2& b) { return a.x == b.x; }), m.end());
    VXA_CUDA(ctx->id_map.ensure(std::max<size_t>(m.size(), 1)));
    if (!m.empty())
        VXA_CUDA(cudaMemcpyAsync(ctx->id_map.ptr, m.data(), m.size() * sizeof(int2), cudaMemcpyHostToDevice,
                                 ctx->stream));
    VXA_CUDA(cudaStreamSynchronize(ctx->stream)); // the host vector goes out of scope
    *map_n = static_cast<uint32_t>(m.size());
    return VXA_OK;
}

// Enqueues one frame. aov/hbo are device buffers or null.
template <typename Real>
int enqueue_frame(vxa_ctx* ctx, const vxa_frame_desc* f, const vxa_instance* in, uint32_t n, PixelAov* aov,
                  HitRec* hbo, vxa_ctx::DeviceHbo* dev_hbo, bool reset_counters) {
    // one upload: the instance records, then (FP32) the float4 cull table,
    // folded straight into the pinned staging slot
    const size_t inst_bytes = (size_t{n} * sizeof(DevInstance<Real>) + 15) & ~size_t{15};
    const size_t cull_bytes = size_t{n} * sizeof(float4); // tile culling (both kernels)
    const size_t bytes = inst_bytes + cull_bytes;
    if (int rc = ensure_staging(ctx, bytes); rc != VXA_OK) return rc;
    const int slot = ctx->inst_slot;
    ctx->inst_slot ^= 1;
    VXA_CUDA(cudaEventSynchronize(ctx->inst_done[slot])); // staging slot no longer read by an earlier copy
    if (ctx->inst_dev[slot].cap < std::max<size_t>(bytes, 16)) {
        VXA_CUDA(cudaEventSynchronize(ctx->inst_free[slot])); // no kernel still reads the old table
        VXA_CUDA(ctx->inst_dev[slot].ensure(std::max<size_t>(bytes, 16)));
    }
    auto* tab = reinterpret_cast<DevInstance<Real>*>(ctx->inst_host[slot]);
    build_instances<Real>(ctx, f, in, n, tab,
                          cull_bytes ? reinterpret_cast<float4*>(ctx->inst_host[slot] + inst_bytes) : nullptr);

    const int32_t W = f->camera.width, H = f->camera.height;
    VXA_CUDA(ctx->fb.ensure(static_cast<size_t>(W) * H));
    ctx->fb_w = W;
    ctx->fb_h = H;
    uint32_t* target = ctx->fb.ptr;
    if (f->tile_world > 1 && ctx->peer_fb != nullptr) {
        if (ctx->peer_w != W || ctx->peer_h != H) return fail(VXA_ERR_INVALID, "peer framebuffer size mismatch");
        target = ctx->peer_fb;
    }

    FrameParams<Real> p{};
    fill_camera(p, f);
    p.inst = reinterpret_cast<const DevInstance<Real>*>(ctx->inst_dev[slot].ptr);
    p.cull = cull_bytes ? reinterpret_cast<const float4*>(ctx->inst_dev[slot].ptr + inst_bytes) : nullptr;
    p.n_inst = n;
    p.background = f->background[0] | (uint32_t{f->background[1]} << 8) | (uint32_t{f->background[2]} << 16) | 0xff000000u;
    p.culling = f->culling ? 1u : 0u;
    p.sorting = f->sorting ? 1u : 0u;
    p.sphere_pass = (f->culling || f->sorting || hbo != nullptr || dev_hbo != nullptr) ? 1u : 0u;
    p.camera_dirty = f->camera_dirty ? 1u : 0u;
    p.rank = f->tile_rank;
    p.world = f->tile_world;
    p.n_super_x = super_tiles_x(W);
    {
        // multiply-high division by n_super_x, exact for every super-tile index
        // s < n_super when s * (magic * n - 2^32) < 2^32; else 0 (plain division)
        const uint64_t n = p.n_super_x, n_super_all = n * static_cast<uint64_t>((H + kSuper - 1) / kSuper);
        const uint64_t m = ((uint64_t{1} << 32) + n - 1) / n, e = m * n - (uint64_t{1} << 32);
        p.super_x_magic = (n > 1 && m < (uint64_t{1} << 32) && (n_super_all - 1) * e < (uint64_t{1} << 32))
                              ? static_cast<uint32_t>(m)
                              : 0u;
    }
    const uint32_t n_super = p.n_super_x * static_cast<uint32_t>((H + kSuper - 1) / kSuper);
    const uint32_t mine = (n_super + static_cast<uint32_t>(f->tile_world - f->tile_rank) - 1) / static_cast<uint32_t>(f->tile_world);
    p.n_tiles = mine * static_cast<uint32_t>(kTilesPerSuper);
    // FrameStats::rays / sphere_tests (renderer.cpp:149-151,253): pixels of this
    // rank's super-tiles, times every object when the sphere pass runs
    uint64_t my_pixels = 0;
    const uint32_t nsy = static_cast<uint32_t>((H + kSuper - 1) / kSuper);
    for (uint32_t sy = 0; sy < nsy; ++sy)
        for (uint32_t sx = 0; sx < p.n_super_x; ++sx)
            if ((sy * p.n_super_x + sx) % static_cast<uint32_t>(f->tile_world) == static_cast<uint32_t>(f->tile_rank))
                my_pixels += static_cast<uint64_t>(std::min<int32_t>(kSuper, W - static_cast<int32_t>(sx) * kSuper)) *
                             static_cast<uint64_t>(std::min<int32_t>(kSuper, H - static_cast<int32_t>(sy) * kSuper));
    ctx->n_rays += my_pixels;
    if (p.sphere_pass) ctx->n_sphere_tests += my_pixels * n;
    p.fb = target;
    p.fence_sys = target != ctx->fb.ptr ? 1u : 0u; // peer stores: fenced before vxa_frame_close's flag
    p.rgb = ctx->next_rgb; // set by vxa_submit_readback for this frame only
    p.band_done = p.rgb != nullptr ? ctx->next_band_done : nullptr;
    p.band_rows = ctx->next_band_rows;
    p.super_done = p.rgb != nullptr ? ctx->next_super_done : nullptr;
    p.rgb_host = p.super_done != nullptr ? ctx->next_rgb_host : nullptr;
    if (p.rgb != nullptr && ctx->next_rgb_free != nullptr) VXA_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->next_rgb_free, 0));
    p.max_depth = 1;
    p.compact = sizeof(Real) == 4 ? 1u : 0u;
    for (uint32_t k = 0; k < n; ++k)
        if (const auto& di = tab[k]; di.valid_model) {
            p.max_depth = std::max(p.max_depth, std::min(di.model.depth, kMaxDepth));
            if (di.model.cwords == nullptr) p.compact = 0;
        }
    // the scene's single model (compact words), whose top node words the FP32
    // kernel stages in shared memory in VXA_SMEM_TOP builds
    p.top_words = nullptr;
    p.top_n = 0;
    if constexpr (sizeof(Real) == 4) {
        const uint32_t* only = nullptr;
        uint32_t nodes = 0;
        bool single = true;
        for (uint32_t k = 0; k < n && single; ++k)
            if (tab[k].valid_model) {
                if (only == nullptr) only = tab[k].model.cwords, nodes = tab[k].model.node_count;
                else if (tab[k].model.cwords != only) single = false;
            }
        if (single && only != nullptr) {
            p.top_words = only;
            p.top_n = std::min<uint32_t>(kSmemTopWords, nodes) & ~3u;
        }
    }
    // VOXANIM_CONTENT_BOUND=off disables the FP32 content-sphere skip (tests: the
    // bound must never change a frame); read per frame
    if (const char* env = std::getenv("VOXANIM_CONTENT_BOUND"); env && std::strcmp(env, "off") == 0)
        for (uint32_t k = 0; k < n; ++k) tab[k].model.content_r2 = 1.0f;
    // VOXANIM_NODE_WORDS=wide forces the general words (tests, A/B timing); read per frame
    if (const char* env = std::getenv("VOXANIM_NODE_WORDS"); env && std::strcmp(env, "wide") == 0) p.compact = 0;
    p.tile_counter = ctx->tile_counter.ptr;
    p.counters = ctx->counters.ptr;
    p.aov = aov;
    p.hbo = hbo;
    p.hbo_compact = 0;
    const size_t npix_hbo = static_cast<size_t>(W) * H;
    // VOXANIM_HBO_COMPACT=0 keeps FP32 frames on the 48-byte records (tests)
    const char* hbo_env = std::getenv("VOXANIM_HBO_COMPACT");
    const bool want_compact = sizeof(Real) == 4 && !(hbo_env && std::strcmp(hbo_env, "0") == 0);
    if (dev_hbo != nullptr && want_compact && dev_hbo->rec16 == nullptr)
        VXA_CUDA(cudaMalloc(&dev_hbo->rec16, npix_hbo * sizeof(HitRec16)));

    // the upload runs beside the previous frame's kernel (its own stream and
    // table slot), off the frame-to-frame critical path
    VXA_CUDA(cudaStreamWaitEvent(ctx->upload_stream, ctx->inst_free[slot], 0));
    if (bytes)
        VXA_CUDA(cudaMemcpyAsync(ctx->inst_dev[slot].ptr, ctx->inst_host[slot], bytes, cudaMemcpyHostToDevice,
                                 ctx->upload_stream));
    ctx->h2d += bytes;
    VXA_CUDA(cudaEventRecord(ctx->inst_done[slot], ctx->upload_stream));
    VXA_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->inst_done[slot], 0));
    // the culling pre-pass (larger scenes) zeroes the work counter and the frame's
    // statistics itself (its first thread): two memset nodes fewer per frame
    const bool prepass = p.culling && n > kSuperCullMin && n <= 0xffffu && p.n_tiles / kTilesPerSuper > 0;
    p.reset_stats = prepass && reset_counters ? 1u : 0u;
    if (!prepass) {
        VXA_CUDA(cudaMemsetAsync(ctx->tile_counter.ptr, 0, sizeof(uint32_t), ctx->stream));
        if (reset_counters)
            VXA_CUDA(cudaMemsetAsync(ctx->counters.ptr, 0, 8 * sizeof(unsigned long long), ctx->stream));
    }

    const bool is64 = sizeof(Real) == 8;
    const bool a = aov != nullptr, h = hbo != nullptr || dev_hbo != nullptr;

    // device hit buffer: bring its records into the format this frame uses
    // (once per switch; both formats describe the same HitRecords)
    if (dev_hbo != nullptr) {
        const unsigned blocks = static_cast<unsigned>((npix_hbo + 255) / 256);
        if (want_compact) {
            if (!dev_hbo->compact) {
                std::vector<int32_t> ids(n);
                for (uint32_t k = 0; k < n; ++k) ids[k] = in[k].id;
                uint32_t map_n = 0;
                if (int rc = upload_id_map(ctx, ids.data(), n, &map_n); rc != VXA_OK) return rc;
                hbo_compress<<<blocks, 256, 0, ctx->stream>>>(dev_hbo->rec, dev_hbo->rec16, npix_hbo,
                                                              reinterpret_cast<const DevInstance<float>*>(p.inst),
                                                              ctx->id_map.ptr, map_n);
                VXA_CUDA(cudaGetLastError());
                dev_hbo->compact = true;
            }
            p.hbo = dev_hbo->rec16;
            p.hbo_compact = 1;
        } else {
            if (dev_hbo->compact) {
                uint32_t map_n = 0;
                if (int rc = upload_id_map(ctx, dev_hbo->tab_ids.data(), dev_hbo->tab_n, &map_n); rc != VXA_OK)
                    return rc;
                hbo_expand<<<blocks, 256, 0, ctx->stream>>>(dev_hbo->rec16, dev_hbo->rec, npix_hbo, dev_hbo->tab.ptr,
                                                            ctx->id_map.ptr, map_n);
                VXA_CUDA(cudaGetLastError());
                dev_hbo->compact = false;
            }
            p.hbo = dev_hbo->rec;
        }
    }
    const int hmode = h ? (p.hbo_compact ? 2 : 1) : 0;
    int& occ = ctx->occ[is64][a][hmode][p.compact][p.max_depth];
    if (occ == 0)
        occ = is64 ? frame_blocks_per_sm_f64(a, hmode, false, p.max_depth)
                   : frame_blocks_per_sm_f32(a, hmode, p.compact, p.max_depth);
    FrameLaunch l{ctx->sm_count * occ, ctx->stream};
    const int slot_k = ctx->k_count % vxa_ctx::kRing;
    if (ctx->k_begin[slot_k] == nullptr) {
        VXA_CUDA(cudaEventCreate(&ctx->k_begin[slot_k]));
        VXA_CUDA(cudaEventCreate(&ctx->k_end[slot_k]));
    }
    VXA_CUDA(cudaEventRecord(ctx->k_begin[slot_k], ctx->stream));
    cudaError_t e = cudaSuccess;
    // larger scenes: per-super-tile candidate lists first (same stream; both kernels)
    if (prepass) {
        const size_t mine_super = p.n_tiles / kTilesPerSuper;
        VXA_CUDA(ctx->super_list.ensure(std::max<size_t>(mine_super * kSuperCap, 1)));
        VXA_CUDA(ctx->super_count.ensure(std::max<size_t>(mine_super, 1)));
        p.super_list = ctx->super_list.ptr;
        p.super_count = ctx->super_count.ptr;
        p.super_cap = kSuperCap;
        if (VXA_TILE_MASKS) { // per-tile candidate masks from the pre-pass
            VXA_CUDA(ctx->tile_mask.ensure(std::max<size_t>(mine_super * kTilesPerSuper, 1)));
            p.tile_mask = ctx->tile_mask.ptr;
        }
        // Longest-first super-tile order (for a banded synchronous readback: bands in
        // screen order, longest-first inside each); VOXANIM_LPT=0 forces screen order
        // (experiments)
        const char* lpt_env = std::getenv("VOXANIM_LPT");
        if (VXA_LPT && !ctx->next_screen_order && !(lpt_env && std::strcmp(lpt_env, "0") == 0)) {
            VXA_CUDA(ctx->super_order.ensure(std::max<size_t>(mine_super, 1)));
            p.super_order = ctx->super_order.ptr;
        }
        e = launch_super_cull(p, ctx->super_list.ptr, ctx->super_count.ptr, ctx->super_done.ptr, ctx->stream);
        ++ctx->aux_launches;
    }
    if (e == cudaSuccess) {
        if constexpr (sizeof(Real) == 8)
            e = launch_frame_f64(p, a, h, l);
        else
            e = launch_frame_f32(p, a, h, l);
    }
    if (e != cudaSuccess) return fail(VXA_ERR_CUDA, std::string("frame kernel launch: ") + cudaGetErrorString(e));
    VXA_CUDA(cudaEventRecord(ctx->k_end[slot_k], ctx->stream));
    if (dev_hbo != nullptr && p.hbo_compact) {
        // the instances the records refer to, for a later expansion (download, FP64 frame)
        VXA_CUDA(dev_hbo->tab.ensure(std::max<size_t>(size_t{9} * n, 9)));
        if (n) hbo_save_table<<<(n + 127) / 128, 128, 0, ctx->stream>>>(
            reinterpret_cast<const DevInstance<float>*>(p.inst), n, dev_hbo->tab.ptr);
        VXA_CUDA(cudaGetLastError());
        dev_hbo->tab_n = n;
        dev_hbo->tab_ids.resize(n);
        for (uint32_t k = 0; k < n; ++k) dev_hbo->tab_ids[k] = in[k].id;
    }
    VXA_CUDA(cudaEventRecord(ctx->inst_free[slot], ctx->stream)); // this table slot may be overwritten now
    ++ctx->k_count;
    return VXA_OK;
}

int enqueue_any(vxa_ctx* ctx, const vxa_frame_desc* f, const vxa_instance* in, uint32_t n, PixelAov* aov, HitRec* hbo,
                vxa_ctx::DeviceHbo* dev_hbo, bool reset) {
    // the FP32 kernel keeps the nearest hit's instance in 24 bits (frame_kernel.cuh: Best<float>)
    if (n >= (1u << 24)) return fail(VXA_ERR_INVALID, "too many instances in one frame (at most 16,777,215)");
    if (f->precision == VXA_FP64) return enqueue_frame<double>(ctx, f, in, n, aov, hbo, dev_hbo, reset);
    return enqueue_frame<float>(ctx, f, in, n, aov, hbo, dev_hbo, reset);
}

// prefetched: the caller already copied the counters into ctx->counters_host
// on the stream and synchronised it (one synchronisation per render call).
int read_counters(vxa_ctx* ctx, vxa_stats* s, bool prefetched = false) {
    unsigned long long c[8] = {};
    if (prefetched && ctx->counters_host != nullptr) {
        std::memcpy(c, ctx->counters_host, sizeof(c));
    } else {
        VXA_CUDA(cudaMemcpyAsync(c, ctx->counters.ptr, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
        VXA_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    s->rays = ctx->n_rays;
    s->sphere_tests = ctx->n_sphere_tests;
    s->svo_traversals = c[2];
    s->pixels_reused = c[3];
    s->node_fetches = c[4];
    s->leaf_hits = c[5];
    // kernel time of the frames since the last reset (the ring keeps the last kRing)
    const int n = std::min(ctx->k_count, vxa_ctx::kRing);
    double total = 0.0;
    for (int i = 0; i < n; ++i) {
        float ms = 0.f;
        VXA_CUDA(cudaEventElapsedTime(&ms, ctx->k_begin[i], ctx->k_end[i]));
        total += ms;
    }
    s->gpu_ms = total;
    s->kernel_launches = static_cast<uint64_t>(ctx->k_count + ctx->aux_launches);
    s->frames = static_cast<uint64_t>(ctx->k_count);
    s->h2d_bytes = ctx->h2d;
    s->d2h_bytes = ctx->d2h + sizeof(c);
    return VXA_OK;
}

} // namespace

// ===========================================================================
// C ABI

extern "C" {

const char* vxa_last_error(void) { return g_error.c_str(); }

int vxa_abi_version(void) { return VXA_ABI_VERSION; }

namespace {
int init_ctx(vxa_ctx* ctx);
}

int vxa_create(int device, vxa_ctx** out) {
    if (out == nullptr) return fail(VXA_ERR_INVALID, "null output pointer");
    *out = nullptr;
    if (device < 0) {
        const char* env = std::getenv("VOXANIM_DEVICE");
        device = env ? std::atoi(env) : 0;
    }
    int count = 0;
    const cudaError_t ce = cudaGetDeviceCount(&count);
    if (ce != cudaSuccess || count == 0)
        return fail(VXA_ERR_NO_DEVICE, std::string("no CUDA device available: ") + cudaGetErrorString(ce));
    if (device >= count) return fail(VXA_ERR_NO_DEVICE, "device ordinal out of range");
    cudaDeviceProp prop{};
    VXA_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(VXA_ERR_NO_DEVICE, std::string("device is not sm_100 (Blackwell): ") + prop.name);
    VXA_CUDA(cudaSetDevice(device));
    auto* ctx = new vxa_ctx;
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    std::snprintf(ctx->name, sizeof(ctx->name), "%s", prop.name);
    if (const int rc = init_ctx(ctx); rc != VXA_OK) {
        vxa_destroy(ctx); // releases whatever was created before the failure
        return rc;
    }
    *out = ctx;
    return VXA_OK;
}

namespace {
// Streams, events and the small device buffers of a new context.
int init_ctx(vxa_ctx* ctx) {
    VXA_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    VXA_CUDA(cudaStreamCreateWithFlags(&ctx->upload_stream, cudaStreamNonBlocking));
    VXA_CUDA(ctx->tile_counter.ensure(1));
    VXA_CUDA(ctx->super_done.ensure(1));
    VXA_CUDA(cudaMemset(ctx->super_done.ptr, 0, sizeof(uint32_t)));
    VXA_CUDA(ctx->counters.ensure(8));
    VXA_CUDA(cudaMemset(ctx->counters.ptr, 0, 8 * sizeof(unsigned long long)));
    for (int s = 0; s < 2; ++s) {
        VXA_CUDA(cudaEventCreateWithFlags(&ctx->inst_done[s], cudaEventDisableTiming));
        VXA_CUDA(cudaEventRecord(ctx->inst_done[s], ctx->upload_stream));
        VXA_CUDA(cudaEventCreateWithFlags(&ctx->inst_free[s], cudaEventDisableTiming));
        VXA_CUDA(cudaEventRecord(ctx->inst_free[s], ctx->stream));
    }
    VXA_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        VXA_CUDA(cudaEventCreateWithFlags(&ctx->rb_packed[k], cudaEventDisableTiming));
        VXA_CUDA(cudaEventCreateWithFlags(&ctx->rb_done[k], cudaEventDisableTiming));
        VXA_CUDA(cudaEventRecord(ctx->rb_done[k], ctx->copy_stream));
    }
    VXA_CUDA(cudaEventCreate(&ctx->ev_a));
    VXA_CUDA(cudaEventCreate(&ctx->ev_b));
    VXA_CUDA(cudaEventCreate(&ctx->t_a));
    VXA_CUDA(cudaEventCreate(&ctx->t_b));
    return VXA_OK;
}
} // namespace

namespace {
int flush_readback(vxa_ctx* ctx);
}

int vxa_destroy(vxa_ctx* ctx) {
    if (ctx == nullptr) return VXA_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) {
        flush_readback(ctx); // a streamed frame still pending lands before teardown
        cudaStreamSynchronize(ctx->stream);
    }
    for (auto& [h, m] : ctx->models) m.free_all();
    ctx->build.grid.release();
    ctx->build.pyramid.release();
    ctx->build.levels.release();
    if (ctx->peer_fb) cudaIpcCloseMemHandle(ctx->peer_fb);
    if (ctx->sync_peer) cudaIpcCloseMemHandle(ctx->sync_peer);
    ctx->sync_own.release();
    ctx->sync_err.release();
    if (ctx->sync_host) cudaFreeHost(ctx->sync_host);
    if (ctx->poll_stream) cudaStreamDestroy(ctx->poll_stream);
    for (auto& [h, b] : ctx->hbos) {
        cudaFree(b.rec);
        cudaFree(b.rec16);
        b.tab.release();
    }
    ctx->fb.release();
    ctx->tile_counter.release();
    ctx->counters.release();
    ctx->inst_dev[0].release();
    ctx->inst_dev[1].release();
    ctx->super_list.release();
    ctx->super_count.release();
    ctx->super_order.release();
    ctx->super_done.release();
    ctx->tile_mask.release();
    ctx->id_map.release();
    ctx->aov.release();
    ctx->hbo.release();
    ctx->rgb.release();
    ctx->l2_scratch.release();
    ctx->band_done.release();
    ctx->direct_done.release();
    if (ctx->band_reset) cudaEventDestroy(ctx->band_reset);
    for (cudaEvent_t e : ctx->band_trace)
        if (e) cudaEventDestroy(e);
    ctx->rays.release();
    ctx->hits.release();
    ctx->visits.release();
    if (ctx->upload_stream) cudaStreamSynchronize(ctx->upload_stream);
    for (int s = 0; s < 2; ++s) {
        if (ctx->inst_host[s]) cudaFreeHost(ctx->inst_host[s]);
        if (ctx->inst_done[s]) cudaEventDestroy(ctx->inst_done[s]);
        if (ctx->inst_free[s]) cudaEventDestroy(ctx->inst_free[s]);
    }
    for (cudaEvent_t e : {ctx->ev_a, ctx->ev_b, ctx->t_a, ctx->t_b})
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < vxa_ctx::kRing; ++i) {
        if (ctx->k_begin[i]) cudaEventDestroy(ctx->k_begin[i]);
        if (ctx->k_end[i]) cudaEventDestroy(ctx->k_end[i]);
    }
    if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
    for (int k = 0; k < 2; ++k) {
        ctx->rb_rgb[k].release();
        if (ctx->rb_packed[k]) cudaEventDestroy(ctx->rb_packed[k]);
        if (ctx->rb_done[k]) cudaEventDestroy(ctx->rb_done[k]);
    }
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->copy_stream2) {
        cudaStreamSynchronize(ctx->copy_stream2);
        cudaStreamDestroy(ctx->copy_stream2);
    }
    if (ctx->upload_stream) cudaStreamDestroy(ctx->upload_stream);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->counters_host) cudaFreeHost(ctx->counters_host);
    delete ctx;
    return VXA_OK;
}

int vxa_device_info(vxa_ctx* ctx, int* device, int* sm_count, char* name, size_t name_len) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (device) *device = ctx->device;
    if (sm_count) *sm_count = ctx->sm_count;
    if (name && name_len) std::snprintf(name, name_len, "%s", ctx->name);
    return VXA_OK;
}

// Radius, in unit-cube coordinates about the cube centre, of a sphere holding
// every leaf: the farthest corner of any leaf, or of any occupied cell of the
// deepest level the walk reaches (a cell bounds its whole subtree). The walk
// goes level by level until a level holds more than kContentCells cells (or the
// caller's node array ends: device-built models pass their top levels only).
// Returned squared with a small margin; the FP32 kernel skips the traversal of
// rays whose line misses it -- a shell's box corners, and the thin annulus
// between the shell and a coarse bound.
#ifndef VXA_CONTENT_CELLS
#define VXA_CONTENT_CELLS 4194304u // cells per level (64 MB of walk state at most)
#endif
// Squared content-sphere radius from the squared farthest leaf extent, with the
// margin the FP32 kernel's test relies on.
float content_bound(double r2) {
    const double rho = std::sqrt(r2) * (1.0 + 1e-5) + 1e-5;
    return static_cast<float>(rho * rho);
}

float content_r2(const uint8_t* raw, uint32_t node_count, uint32_t depth) {
    const int K = static_cast<int>(depth);
    constexpr size_t kContentCells = VXA_CONTENT_CELLS;
    struct Cell {
        uint32_t idx, x, y, z;
    };
    std::vector<Cell> cur{{0, 0, 0, 0}}, next;
    double r2 = 0.0;
    const auto corner2 = [](uint32_t x, uint32_t y, uint32_t z, int L) {
        const double sz = std::ldexp(1.0, -L);
        double acc = 0.0;
        for (const uint32_t c : {x, y, z}) {
            const double lo = c * sz - 0.5, hi = (c + 1) * sz - 0.5;
            acc += std::max(lo * lo, hi * hi);
        }
        return acc;
    };
    for (int L = 0; L < K; ++L) {
        bool inside = true;
        for (const Cell& c : cur) inside = inside && c.idx < node_count;
        if (!inside) { // the nodes below are not here (top levels only): bound by the cells
            for (const Cell& c : cur) r2 = std::max(r2, corner2(c.x, c.y, c.z, L));
            break;
        }
        next.clear();
        bool full = false;
        for (const Cell& c : cur) {
            const uint8_t* r = raw + 12 * size_t{c.idx};
            uint32_t cb;
            std::memcpy(&cb, r, 4);
            const uint32_t valid = r[8], leaf = r[9], internal = valid & ~leaf & 0xffu;
            for (uint32_t o = 0; o < 8; ++o) {
                if (!((valid >> o) & 1u)) continue;
                const uint32_t x = 2 * c.x + ((o >> 2) & 1u), y = 2 * c.y + ((o >> 1) & 1u), z = 2 * c.z + (o & 1u);
                if (((leaf >> o) & 1u) || L + 1 == K)
                    r2 = std::max(r2, corner2(x, y, z, L + 1));
                else
                    next.push_back({cb + static_cast<uint32_t>(__builtin_popcount(internal & ((1u << o) - 1u))), x, y, z});
            }
            if (next.size() > kContentCells) {
                full = true;
                break;
            }
        }
        if (full) { // the next level would not fit: bound by this level's cells
            for (const Cell& c : cur) r2 = std::max(r2, corner2(c.x, c.y, c.z, L));
            break;
        }
        cur.swap(next);
    }
    return content_bound(r2);
}

int vxa_upload_model(vxa_ctx* ctx, const void* nodes, uint32_t node_count, const void* attrs, uint32_t attr_count,
                     uint32_t depth, uint32_t* handle_out) {
    if (ctx == nullptr || handle_out == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (nodes == nullptr || node_count == 0) return fail(VXA_ERR_MODEL, "model has no root node");
    if (depth < 1 || depth > kMaxDepth) return fail(VXA_ERR_MODEL, "depth out of range [1, 16]");
    if (attr_count > 0 && attrs == nullptr) return fail(VXA_ERR_INVALID, "null attribute array");
    VXA_CUDA(cudaSetDevice(ctx->device));
    // reference validate() rules (svo.cpp:134-172)
    const auto* raw = static_cast<const uint8_t*>(nodes);
    bool any_mixed = false;
    for (uint32_t i = 0; i < node_count; ++i) {
        uint32_t cb, ab;
        std::memcpy(&cb, raw + 12 * size_t{i}, 4);
        std::memcpy(&ab, raw + 12 * size_t{i} + 4, 4);
        const uint32_t valid = raw[12 * size_t{i} + 8], leaf = raw[12 * size_t{i} + 9];
        if (leaf & ~valid) return fail(VXA_ERR_MODEL, "node " + std::to_string(i) + ": leaf_mask outside valid_mask");
        const uint32_t internal = valid & ~leaf & 0xffu, leaves = valid & leaf;
        const int ni = __builtin_popcount(internal), nl = __builtin_popcount(leaves);
        if (ni > 0 && (uint64_t{cb} + ni > node_count || cb <= i))
            return fail(VXA_ERR_MODEL, "node " + std::to_string(i) + ": child_base out of range");
        if (nl > 0 && uint64_t{ab} + nl > attr_count)
            return fail(VXA_ERR_MODEL, "node " + std::to_string(i) + ": attr_base out of range");
        any_mixed |= ni > 0 && nl > 0;
    }
    // Canonical models (leaves exactly at the last level, bases < 2^24) also get
    // compact 4-byte words: valid | base << 8. Levels follow from the BFS-free
    // rule "children come after their parent" (validated above).
    std::vector<uint32_t> compact;
    {
        std::vector<uint8_t> lvl(node_count, 0);
        bool ok = node_count < (1u << 24) && attr_count <= (1u << 24);
        for (uint32_t i = 0; i < node_count && ok; ++i) {
            const uint8_t* r = raw + 12 * size_t{i};
            uint32_t cb, ab;
            std::memcpy(&cb, r, 4);
            std::memcpy(&ab, r + 4, 4);
            const uint32_t valid = r[8], leaf = r[9];
            const uint32_t internal = valid & ~leaf & 0xffu;
            const bool last = lvl[i] + 1u == depth;
            if (last ? (leaf != valid) : (leaf != 0)) ok = false;
            if (internal) {
                const int ni = __builtin_popcount(internal);
                for (int k = 0; k < ni; ++k) lvl[cb + k] = static_cast<uint8_t>(lvl[i] + 1);
            }
            if (ok) {
                const uint32_t base = last ? ab : cb;
                if (base >= (1u << 24)) ok = false;
                compact.push_back(valid | ((valid ? base : 0u) << 8));
            }
        }
        if (!ok) compact.clear();
    }
    ModelEntry m;
    uint32_t* raw_dev = nullptr;
    const size_t raw_bytes = 12 * size_t{node_count};
    VXA_CUDA(cudaMalloc(&raw_dev, raw_bytes));
    cudaError_t e = cudaMalloc(&m.words, sizeof(uint2) * node_count);
    if (e == cudaSuccess && any_mixed) e = cudaMalloc(&m.side, sizeof(uint32_t) * node_count);
    if (e == cudaSuccess) e = cudaMalloc(&m.attrs, sizeof(uint32_t) * std::max<uint32_t>(attr_count, 1));
    if (e == cudaSuccess && !compact.empty()) e = cudaMalloc(&m.cwords, sizeof(uint32_t) * node_count);
    if (e == cudaSuccess && !compact.empty())
        e = cudaMemcpyAsync(m.cwords, compact.data(), sizeof(uint32_t) * node_count, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(raw_dev, nodes, raw_bytes, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess && attr_count)
        e = cudaMemcpyAsync(m.attrs, attrs, sizeof(uint32_t) * attr_count, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) {
        repack_nodes<<<(node_count + 255) / 256, 256, 0, ctx->stream>>>(raw_dev, node_count, m.words, m.side);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    m.raw = raw_dev;
    if (e != cudaSuccess) {
        m.free_all();
        return fail(e == cudaErrorMemoryAllocation ? VXA_ERR_OOM : VXA_ERR_CUDA,
                    std::string("model upload: ") + cudaGetErrorString(e));
    }
    m.dev.words = m.words;
    m.dev.cwords = m.cwords;
    m.dev.side = m.side;
    m.dev.attrs = m.attrs;
    m.dev.depth = depth;
    m.dev.node_count = node_count;
    m.dev.content_r2 = content_r2(raw, node_count, depth);
    m.attr_count = attr_count;
    m.bytes = sizeof(uint2) * uint64_t{node_count} + (any_mixed ? 4ull * node_count : 0) + 4ull * attr_count +
              (m.cwords ? 4ull * node_count : 0) + raw_bytes;
    const uint32_t handle = ctx->next_handle++;
    ctx->models[handle] = m;
    *handle_out = handle;
    return VXA_OK;
}

int vxa_upload_svo(vxa_ctx* ctx, const uint8_t* bytes, size_t size, uint32_t* handle_out, int32_t* format_error) {
    if (format_error) *format_error = -1;
    if (ctx == nullptr || handle_out == nullptr || (bytes == nullptr && size > 0))
        return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    const auto bad = [&](int code, const std::string& msg) {
        if (format_error) *format_error = code;
        return fail(VXA_ERR_MODEL, msg);
    };
    const auto u32 = [&](size_t off) {
        return uint32_t{bytes[off]} | (uint32_t{bytes[off + 1]} << 8) | (uint32_t{bytes[off + 2]} << 16) |
               (uint32_t{bytes[off + 3]} << 24);
    };
    // deserialize()'s checks, in its order (svo.cpp:232-258)
    constexpr size_t kHeader = 20;
    if (size < kHeader) return bad(3, "svo: truncated header");
    if (std::memcmp(bytes, "SVOA", 4) != 0) return bad(0, "svo: bad magic, not an SVOA file");
    if (u32(4) != 1) return bad(1, "svo: unsupported version " + std::to_string(u32(4)));
    const uint32_t depth = u32(8), node_count = u32(12), attr_count = u32(16);
    if (depth < 1 || depth > kMaxDepth || node_count == 0)
        return bad(2, "svo: bad header (depth or node count out of range)");
    const size_t expected = kHeader + 12 * size_t{node_count} + 4 * size_t{attr_count};
    if (size < expected) return bad(3, "svo: truncated payload");
    if (size > expected) return bad(4, "svo: trailing bytes after payload");
    const uint8_t* nodes = bytes + kHeader;
    for (uint32_t i = 0; i < node_count; ++i) {
        const uint8_t* r = nodes + 12 * size_t{i};
        const uint32_t valid = r[8], leaf = r[9];
        const int ni = __builtin_popcount(valid & ~leaf & 0xffu), nl = __builtin_popcount(valid & leaf);
        uint32_t cb, ab;
        std::memcpy(&cb, r, 4);
        std::memcpy(&ab, r + 4, 4);
        if (ni > 0 && uint64_t{cb} + ni > node_count)
            return bad(5, "svo: node " + std::to_string(i) + " child_base out of range");
        if (nl > 0 && uint64_t{ab} + nl > attr_count)
            return bad(6, "svo: node " + std::to_string(i) + " attr_base out of range");
    }
    // the stream's node records are the 12-byte SvoNode layout (little endian)
    return vxa_upload_model(ctx, nodes, node_count, nodes + 12 * size_t{node_count}, attr_count, depth, handle_out);
}

int vxa_release_model(vxa_ctx* ctx, uint32_t handle) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    const auto it = ctx->models.find(handle);
    if (it == ctx->models.end()) return fail(VXA_ERR_INVALID, "unknown model handle");
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    it->second.free_all();
    ctx->models.erase(it);
    return VXA_OK;
}

int vxa_model_info(vxa_ctx* ctx, uint32_t handle, uint64_t* device_bytes, uint32_t* node_format) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    const auto it = ctx->models.find(handle);
    if (it == ctx->models.end()) return fail(VXA_ERR_INVALID, "unknown model handle");
    if (device_bytes) *device_bytes = it->second.bytes;
    if (node_format) *node_format = it->second.cwords ? 1 : 2;
    return VXA_OK;
}

int vxa_build_model(vxa_ctx* ctx, const uint64_t* grid_words, uint32_t depth, uint32_t color_mode,
                    uint32_t color_rgba, uint32_t* handle_out, uint64_t* node_count, uint64_t* attr_count) {
    if (ctx == nullptr || handle_out == nullptr || grid_words == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    // build_from_grid's argument checks (svo.cpp:80-87) plus the dense-grid cap (ingest.cpp:15)
    if (depth < 1 || depth > 10) return fail(VXA_ERR_INVALID, "octree depth must be in [1, 10] for a dense grid");
    if (color_mode > 2) return fail(VXA_ERR_INVALID, "unknown colour mode");
    VXA_CUDA(cudaSetDevice(ctx->device));
    const uint64_t n = uint64_t{1} << depth;
    const size_t grid_bytes = 8 * ((n * n * n + 63) / 64);
    VXA_CUDA(ctx->build.grid.ensure(grid_bytes));
    auto* grid_dev = static_cast<uint64_t*>(ctx->build.grid.p);
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaMemcpyAsync(grid_dev, grid_words, grid_bytes, cudaMemcpyHostToDevice, ctx->stream);
    if (std::getenv("VOXANIM_BUILD_TRACE")) {
        cudaStreamSynchronize(ctx->stream);
        std::fprintf(stderr, "[build] grid H2D     %8.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    BuiltModel b;
    if (e == cudaSuccess) e = build_svo(ctx->stream, grid_dev, depth, color_mode, color_rgba, ctx->build, b);
    ModelEntry m;
    m.block = b.block;
    m.raw = b.records;
    m.attrs = b.attrs;
    m.cwords = b.cwords;
    m.words = b.words;
    if (e == cudaSuccess) {
        // canonical by construction: no mixed nodes, so no side table
        repack_nodes<<<static_cast<unsigned>((b.node_count + 255) / 256), 256, 0, ctx->stream>>>(
            m.raw, static_cast<uint32_t>(b.node_count), m.words, nullptr);
        e = cudaGetLastError();
    }
    // the builder's leaf extent (content bound, below): read under the same synchronisation
    if (e == cudaSuccess && ctx->counters_host == nullptr)
        e = cudaMallocHost(&ctx->counters_host, 8 * sizeof(unsigned long long));
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(ctx->counters_host, b.extent_dev, sizeof(unsigned int), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        cudaStreamSynchronize(ctx->stream);
        m.free_all();
        if (e == cudaErrorInvalidValue) return fail(VXA_ERR_MODEL, "model exceeds 2^32 nodes or attributes");
        return fail(e == cudaErrorMemoryAllocation ? VXA_ERR_OOM : VXA_ERR_CUDA,
                    std::string("device model build: ") + cudaGetErrorString(e));
    }
    m.dev.words = m.words;
    m.dev.cwords = m.cwords;
    m.dev.side = nullptr;
    m.dev.attrs = m.attrs;
    m.dev.depth = depth;
    m.dev.node_count = static_cast<uint32_t>(b.node_count);
    {
        // content bound: the farthest leaf corner, reduced on the device by the builder
        unsigned int bits = 0;
        std::memcpy(&bits, ctx->counters_host, sizeof(bits));
        float r2;
        std::memcpy(&r2, &bits, sizeof(r2));
        m.dev.content_r2 = content_bound(static_cast<double>(r2));
    }
    m.attr_count = b.attr_count;
    m.bytes = (8 + 12 + (m.cwords ? 4 : 0)) * b.node_count + 4 * b.attr_count;
    const uint32_t handle = ctx->next_handle++;
    ctx->models[handle] = m;
    *handle_out = handle;
    if (node_count) *node_count = b.node_count;
    if (attr_count) *attr_count = b.attr_count;
    return VXA_OK;
}

int vxa_model_download(vxa_ctx* ctx, uint32_t handle, void* nodes, uint64_t node_cap, uint32_t* attrs,
                       uint64_t attr_cap) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    const auto it = ctx->models.find(handle);
    if (it == ctx->models.end()) return fail(VXA_ERR_INVALID, "unknown model handle");
    const ModelEntry& m = it->second;
    if ((nodes && node_cap < m.dev.node_count) || (attrs && attr_cap < m.attr_count))
        return fail(VXA_ERR_INVALID, "output arrays too small");
    VXA_CUDA(cudaSetDevice(ctx->device));
    if (nodes) VXA_CUDA(cudaMemcpyAsync(nodes, m.raw, 12 * uint64_t{m.dev.node_count}, cudaMemcpyDeviceToHost, ctx->stream));
    if (attrs && m.attr_count)
        VXA_CUDA(cudaMemcpyAsync(attrs, m.attrs, 4 * m.attr_count, cudaMemcpyDeviceToHost, ctx->stream));
    VXA_CUDA(cudaStreamSynchronize(ctx->stream));
    return VXA_OK;
}

int vxa_model_counts(vxa_ctx* ctx, uint32_t handle, uint32_t* depth, uint64_t* node_count, uint64_t* attr_count) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    const auto it = ctx->models.find(handle);
    if (it == ctx->models.end()) return fail(VXA_ERR_INVALID, "unknown model handle");
    if (depth) *depth = it->second.dev.depth;
    if (node_count) *node_count = it->second.dev.node_count;
    if (attr_count) *attr_count = it->second.attr_count;
    return VXA_OK;
}

namespace {
// cuStreamWaitValue32 through the runtime's driver entry point (no libcuda link);
// VOXANIM_BANDED_READBACK=0 turns the banded synchronous readback off.
bool band_api_ok(vxa_ctx* ctx) {
    if (const char* env = std::getenv("VOXANIM_BANDED_READBACK"); env && std::strcmp(env, "0") == 0) return false;
    if (ctx->band_api == 0) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        ctx->band_api = (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
                         q == cudaDriverEntryPointSuccess && fn != nullptr)
                            ? 1
                            : -1;
        ctx->wait_value32 = fn;
        cudaGetLastError();
    }
    return ctx->band_api > 0;
}
} // namespace

int vxa_render(vxa_ctx* ctx, const vxa_frame_desc* f, const vxa_instance* in, uint32_t n, uint8_t* rgb_out,
               vxa_pixel_aov* aov_out, vxa_stats* stats) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (int rc = check_frame(f); rc != VXA_OK) return rc;
    if (n > 0 && in == nullptr) return fail(VXA_ERR_INVALID, "null instance array");
    VXA_CUDA(cudaSetDevice(ctx->device));
    const size_t npix = static_cast<size_t>(f->camera.width) * f->camera.height;
    PixelAov* aov = nullptr;
    HitRec* hbo = nullptr;
    if (aov_out) {
        VXA_CUDA(ctx->aov.ensure(npix));
        aov = ctx->aov.ptr;
        VXA_CUDA(cudaMemsetAsync(aov, 0, npix * sizeof(PixelAov), ctx->stream));
    }
    if (f->hbo && f->hbo_device) return fail(VXA_ERR_INVALID, "host and device hit buffers are exclusive");
    vxa_ctx::DeviceHbo* dev_hbo = nullptr;
    if (f->hbo_device) {
        const auto it = ctx->hbos.find(f->hbo_device);
        if (it == ctx->hbos.end()) return fail(VXA_ERR_INVALID, "unknown hit buffer handle");
        if (it->second.w != f->camera.width || it->second.h != f->camera.height)
            return fail(VXA_ERR_INVALID, "hit buffer dimensions do not match the camera");
        dev_hbo = &it->second;
    }
    if (f->hbo) {
        VXA_CUDA(ctx->hbo.ensure(npix));
        hbo = ctx->hbo.ptr;
        VXA_CUDA(cudaMemcpyAsync(hbo, f->hbo, npix * sizeof(HitRec), cudaMemcpyHostToDevice, ctx->stream));
        ctx->h2d += npix * sizeof(HitRec);
    }
    ctx->k_count = 0;
    ctx->aux_launches = 0;
    ctx->h2d = ctx->d2h = 0;
    ctx->n_rays = ctx->n_sphere_tests = 0;
    VXA_CUDA(cudaEventRecord(ctx->ev_a, ctx->stream));
    // the frame kernel writes the RGB8 image itself for an unpartitioned frame
    // (this call is synchronous, so the buffer is free: no wait event)
    const bool fused = rgb_out != nullptr && f->tile_world == 1;
    // Large frames: the RGB8 image goes to the host in bands of super-tile rows,
    // each band's D2H on the copy stream as soon as the frame kernel has finished
    // its tiles (a stream wait on the band's tile counter), overlapping the rest
    // of the frame; the last band's copy is all that follows the kernel.
    const uint32_t n_sx = super_tiles_x(f->camera.width);
    const uint32_t n_sy = static_cast<uint32_t>((f->camera.height + kSuper - 1) / kSuper);
    // Direct mode: when the caller's image is page-locked and mapped (vxa_host_register,
    // cudaHostAlloc), the warp finishing a super-tile stores its rows straight into it
    // over PCIe (frame_kernel.cuh: flush_super_rgb), so the transfer runs alongside
    // the frame from its first finished super-tile on and only the last one's rows
    // follow the kernel. VOXANIM_DIRECT_READBACK=0 turns it off.
    uint8_t* direct_host = nullptr;
    if (fused && npix >= (size_t{1} << 20) && aov_out == nullptr && hbo == nullptr && dev_hbo == nullptr) {
        const char* env = std::getenv("VOXANIM_DIRECT_READBACK");
        if (!(env && std::strcmp(env, "0") == 0)) {
            cudaPointerAttributes a{};
            if (cudaPointerGetAttributes(&a, rgb_out) == cudaSuccess && a.type == cudaMemoryTypeHost &&
                a.devicePointer != nullptr)
                direct_host = static_cast<uint8_t*>(a.devicePointer);
            cudaGetLastError();
        }
    }
    uint32_t band_rows = 0, n_bands = 0;
    if (fused && direct_host == nullptr && npix >= (size_t{1} << 20) && band_api_ok(ctx)) {
        // about VOXANIM_READBACK_BANDS bands (default 16, at most 16: the frame kernel's band counters)
        uint32_t want = 16;
        if (const char* env = std::getenv("VOXANIM_READBACK_BANDS"); env && std::atoi(env) > 0)
            want = std::min<uint32_t>(16, static_cast<uint32_t>(std::atoi(env)));
        band_rows = (n_sy + want - 1) / want;
        n_bands = (n_sy + band_rows - 1) / band_rows;
    }
    if (fused) {
        VXA_CUDA(ctx->rgb.ensure(npix * 3 + 16));
        ctx->next_rgb = ctx->rgb.ptr;
        ctx->next_rgb_free = nullptr;
    }
    if (n_bands) {
        VXA_CUDA(ctx->band_done.ensure(16));
        VXA_CUDA(cudaMemsetAsync(ctx->band_done.ptr, 0, 16 * sizeof(uint32_t), ctx->stream));
        if (ctx->band_reset == nullptr) VXA_CUDA(cudaEventCreateWithFlags(&ctx->band_reset, cudaEventDisableTiming));
        VXA_CUDA(cudaEventRecord(ctx->band_reset, ctx->stream));
        if (int rc = flush_readback(ctx); rc != VXA_OK) return rc;
        VXA_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->band_reset, 0)); // no wait sees last frame's counts
        if (ctx->copy_stream2 == nullptr) VXA_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream2, cudaStreamNonBlocking));
        VXA_CUDA(cudaStreamWaitEvent(ctx->copy_stream2, ctx->band_reset, 0));
        ctx->next_band_done = ctx->band_done.ptr;
        ctx->next_band_rows = band_rows;
    }
    if (direct_host) {
        const size_t n_super = static_cast<size_t>(n_sx) * n_sy;
        VXA_CUDA(ctx->direct_done.ensure(n_super));
        VXA_CUDA(cudaMemsetAsync(ctx->direct_done.ptr, 0, n_super * sizeof(uint32_t), ctx->stream));
        ctx->next_super_done = ctx->direct_done.ptr;
        ctx->next_rgb_host = direct_host;
        // super-tile order (VOXANIM_DIRECT_ORDER): screen order (default: the finished
        // super-tiles and their PCIe stores spread over the frame), longest-first ("lpt":
        // the cheap super-tiles finish in a burst at the end and their stores queue
        // behind the kernel), or banded ("banded": 16 bands in screen order,
        // longest-first inside each)
        const char* ord = std::getenv("VOXANIM_DIRECT_ORDER");
        const std::string order = ord ? ord : "screen";
        ctx->next_screen_order = order == "screen";
        if (order == "banded") ctx->next_band_rows = (n_sy + 15) / 16;
    }
    const int erc = enqueue_any(ctx, f, in, n, aov, hbo, dev_hbo, true);
    ctx->next_rgb = nullptr;
    ctx->next_band_done = nullptr;
    ctx->next_band_rows = 0;
    ctx->next_super_done = nullptr;
    ctx->next_rgb_host = nullptr;
    ctx->next_screen_order = false;
    if (erc != VXA_OK) return erc;
    VXA_CUDA(cudaEventRecord(ctx->ev_b, ctx->stream));
    uint64_t launches = 1 + static_cast<uint64_t>(ctx->aux_launches);
    if (rgb_out && fused && n_bands) {
        // VOXANIM_BAND_TRACE=1: per-band copy completion times relative to the frame (stderr)
        static const bool trace = [] {
            const char* e = std::getenv("VOXANIM_BAND_TRACE");
            return e && std::strcmp(e, "1") == 0;
        }();
        cudaEvent_t* const trace_ev = ctx->band_trace;
        if (trace && trace_ev[0] == nullptr)
            for (int b = 0; b < 16; ++b) VXA_CUDA(cudaEventCreate(&trace_ev[b]));
        using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
        const auto wait = reinterpret_cast<WaitFn>(ctx->wait_value32);
        const size_t row_bytes = static_cast<size_t>(f->camera.width) * 3;
        // bands alternate between two copy streams (two DMA engines: one D2H stream
        // alone reaches ~45 GB/s on these band sizes); VOXANIM_READBACK_STREAMS=1: one
        const char* ns_env = std::getenv("VOXANIM_READBACK_STREAMS");
        const bool two = !(ns_env && std::strcmp(ns_env, "1") == 0);
        for (uint32_t b = 0; b < n_bands; ++b) {
            const uint32_t r0 = b * band_rows, r1 = std::min(n_sy, r0 + band_rows);
            const uint32_t tiles = (r1 - r0) * n_sx * static_cast<uint32_t>(kTilesPerSuper);
            cudaStream_t cs = (two && (b & 1u)) ? ctx->copy_stream2 : ctx->copy_stream;
            const CUresult cr = wait(reinterpret_cast<CUstream>(cs),
                                     reinterpret_cast<CUdeviceptr>(ctx->band_done.ptr + b), tiles,
                                     CU_STREAM_WAIT_VALUE_GEQ);
            if (cr != CUDA_SUCCESS) return fail(VXA_ERR_CUDA, "cuStreamWaitValue32 failed");
            const size_t y0 = static_cast<size_t>(r0) * kSuper;
            const size_t y1 = std::min<size_t>(static_cast<size_t>(r1) * kSuper, static_cast<size_t>(f->camera.height));
            VXA_CUDA(cudaMemcpyAsync(rgb_out + y0 * row_bytes, ctx->rgb.ptr + y0 * row_bytes, (y1 - y0) * row_bytes,
                                     cudaMemcpyDeviceToHost, cs));
            if (trace) VXA_CUDA(cudaEventRecord(trace_ev[b], cs));
        }
        ctx->d2h += npix * 3;
        if (trace) {
            VXA_CUDA(cudaStreamSynchronize(ctx->copy_stream));
            VXA_CUDA(cudaStreamSynchronize(ctx->copy_stream2));
            VXA_CUDA(cudaStreamSynchronize(ctx->stream));
            float k = 0.f;
            cudaEventElapsedTime(&k, ctx->ev_a, ctx->ev_b);
            std::fprintf(stderr, "band trace: frame end %.3f ms; band copies done at", k);
            for (uint32_t b = 0; b < n_bands; ++b) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, ctx->ev_a, trace_ev[b]);
                std::fprintf(stderr, " %.3f", ms);
            }
            std::fprintf(stderr, "\n");
        }
    } else if (rgb_out && fused && direct_host) {
        ctx->d2h += npix * 3; // stored by the frame kernel; visible once the stream is synchronised
    } else if (rgb_out && fused) {
        VXA_CUDA(cudaMemcpyAsync(rgb_out, ctx->rgb.ptr, npix * 3, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->d2h += npix * 3;
    } else if (rgb_out) {
        VXA_CUDA(ctx->rgb.ensure(npix * 3 + 16));
        const size_t quads = (npix + 3) / 4;
        pack_rgb<<<static_cast<unsigned>((quads + 255) / 256), 256, 0, ctx->stream>>>(ctx->fb.ptr, ctx->rgb.ptr, npix);
        VXA_CUDA(cudaGetLastError());
        ++launches;
        VXA_CUDA(cudaMemcpyAsync(rgb_out, ctx->rgb.ptr, npix * 3, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->d2h += npix * 3;
    }
    if (aov_out) {
        VXA_CUDA(cudaMemcpyAsync(aov_out, aov, npix * sizeof(PixelAov), cudaMemcpyDeviceToHost, ctx->stream));
        ctx->d2h += npix * sizeof(PixelAov);
    }
    if (f->hbo) {
        VXA_CUDA(cudaMemcpyAsync(f->hbo, hbo, npix * sizeof(HitRec), cudaMemcpyDeviceToHost, ctx->stream));
        ctx->d2h += npix * sizeof(HitRec);
    }
    if (stats) { // counters ride the same synchronisation as the image
        if (ctx->counters_host == nullptr)
            VXA_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->counters_host), 8 * sizeof(unsigned long long),
                                   cudaHostAllocDefault));
        VXA_CUDA(cudaMemcpyAsync(ctx->counters_host, ctx->counters.ptr, 8 * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, ctx->stream));
    }
    VXA_CUDA(cudaStreamSynchronize(ctx->stream));
    if (n_bands) {
        VXA_CUDA(cudaStreamSynchronize(ctx->copy_stream));
        VXA_CUDA(cudaStreamSynchronize(ctx->copy_stream2));
    }
    if (stats) {
        if (int rc = read_counters(ctx, stats, true); rc != VXA_OK) return rc;
        stats->kernel_launches = launches;
    }
    return VXA_OK;
}

int vxa_hbo_create(vxa_ctx* ctx, int32_t width, int32_t height, uint32_t* handle_out) {
    if (ctx == nullptr || handle_out == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (width < 1 || height < 1) return fail(VXA_ERR_INVALID, "bad hit buffer size");
    VXA_CUDA(cudaSetDevice(ctx->device));
    const size_t n = static_cast<size_t>(width) * height;
    vxa_ctx::DeviceHbo b;
    VXA_CUDA(cudaMalloc(&b.rec, n * sizeof(HitRec)));
    b.w = width;
    b.h = height;
    init_hit_records<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(b.rec, n);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        cudaFree(b.rec);
        return fail(VXA_ERR_CUDA, std::string("hbo init: ") + cudaGetErrorString(e));
    }
    const uint32_t h = ctx->next_hbo++;
    ctx->hbos[h] = b;
    *handle_out = h;
    return VXA_OK;
}

int vxa_hbo_release(vxa_ctx* ctx, uint32_t handle) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    const auto it = ctx->hbos.find(handle);
    if (it == ctx->hbos.end()) return fail(VXA_ERR_INVALID, "unknown hit buffer handle");
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(it->second.rec);
    cudaFree(it->second.rec16);
    it->second.tab.release();
    ctx->hbos.erase(it);
    return VXA_OK;
}

int vxa_hbo_download(vxa_ctx* ctx, uint32_t handle, vxa_hit_record* out) {
    if (ctx == nullptr || out == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    const auto it = ctx->hbos.find(handle);
    if (it == ctx->hbos.end()) return fail(VXA_ERR_INVALID, "unknown hit buffer handle");
    VXA_CUDA(cudaSetDevice(ctx->device));
    const size_t n = static_cast<size_t>(it->second.w) * it->second.h;
    const HitRec* src = it->second.rec;
    if (it->second.compact) { // FP32 frames left 16-byte records: expand them (the buffer stays compact)
        VXA_CUDA(ctx->hbo.ensure(n));
        uint32_t map_n = 0;
        if (int rc = upload_id_map(ctx, it->second.tab_ids.data(), it->second.tab_n, &map_n); rc != VXA_OK) return rc;
        hbo_expand<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(
            it->second.rec16, ctx->hbo.ptr, n, it->second.tab.ptr, ctx->id_map.ptr, map_n);
        VXA_CUDA(cudaGetLastError());
        src = ctx->hbo.ptr;
    }
    VXA_CUDA(cudaMemcpyAsync(out, src, n * sizeof(HitRec), cudaMemcpyDeviceToHost, ctx->stream));
    VXA_CUDA(cudaStreamSynchronize(ctx->stream));
    return VXA_OK;
}

int vxa_hbo_upload(vxa_ctx* ctx, uint32_t handle, const vxa_hit_record* in) {
    if (ctx == nullptr || in == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    const auto it = ctx->hbos.find(handle);
    if (it == ctx->hbos.end()) return fail(VXA_ERR_INVALID, "unknown hit buffer handle");
    VXA_CUDA(cudaSetDevice(ctx->device));
    const size_t n = static_cast<size_t>(it->second.w) * it->second.h;
    VXA_CUDA(cudaMemcpyAsync(it->second.rec, in, n * sizeof(HitRec), cudaMemcpyHostToDevice, ctx->stream));
    VXA_CUDA(cudaStreamSynchronize(ctx->stream));
    it->second.compact = false; // the next FP32 frame compresses the uploaded records
    ctx->h2d += n * sizeof(HitRec);
    return VXA_OK;
}

int vxa_submit(vxa_ctx* ctx, const vxa_frame_desc* f, const vxa_instance* in, uint32_t n) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (int rc = check_frame(f); rc != VXA_OK) return rc;
    if (f->hbo) return fail(VXA_ERR_INVALID, "vxa_submit does not take a host hit buffer");
    if (n > 0 && in == nullptr) return fail(VXA_ERR_INVALID, "null instance array");
    VXA_CUDA(cudaSetDevice(ctx->device));
    vxa_ctx::DeviceHbo* dev_hbo = nullptr;
    if (f->hbo_device) {
        const auto it = ctx->hbos.find(f->hbo_device);
        if (it == ctx->hbos.end()) return fail(VXA_ERR_INVALID, "unknown hit buffer handle");
        if (it->second.w != f->camera.width || it->second.h != f->camera.height)
            return fail(VXA_ERR_INVALID, "hit buffer dimensions do not match the camera");
        dev_hbo = &it->second;
    }
    return enqueue_any(ctx, f, in, n, nullptr, nullptr, dev_hbo, false);
}

namespace {
// Enqueues the deferred D2H of the newest streamed frame (caller holds ctx->mu).
int flush_readback(vxa_ctx* ctx) {
    if (!ctx->rb_pending) return VXA_OK;
    const int slot = ctx->rb_pending_slot;
    ctx->rb_pending = false;
    VXA_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->rb_packed[slot], 0));
    VXA_CUDA(cudaMemcpyAsync(ctx->rb_pending_out, ctx->rb_rgb[slot].ptr, ctx->rb_pending_bytes, cudaMemcpyDeviceToHost,
                             ctx->copy_stream));
    VXA_CUDA(cudaEventRecord(ctx->rb_done[slot], ctx->copy_stream));
    return VXA_OK;
}
} // namespace

int vxa_submit_readback(vxa_ctx* ctx, const vxa_frame_desc* f, const vxa_instance* in, uint32_t n,
                        uint8_t* rgb_out, uint64_t* ticket) {
    if (ctx == nullptr || rgb_out == nullptr || ticket == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (int rc = check_frame(f); rc != VXA_OK) return rc;
    const size_t npix = static_cast<size_t>(f->camera.width) * f->camera.height;
    const int slot = static_cast<int>(ctx->rb_next & 1u);
    VXA_CUDA(ctx->rb_rgb[slot].ensure(npix * 3 + 16));
    // The frame kernel writes the RGB8 bytes into the slot itself (no pack
    // pass), after the slot's previous D2H (two frames back) is done.
    ctx->next_rgb = f->tile_world == 1 ? ctx->rb_rgb[slot].ptr : nullptr;
    ctx->next_rgb_free = ctx->rb_done[slot];
    const int rc = vxa_submit(ctx, f, in, n);
    const bool fused = ctx->next_rgb != nullptr;
    ctx->next_rgb = nullptr;
    if (rc != VXA_OK) return rc;
    if (!fused) { // a partitioned frame: pack the composed framebuffer
        VXA_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->rb_done[slot], 0));
        const size_t quads = (npix + 3) / 4;
        pack_rgb<<<static_cast<unsigned>((quads + 255) / 256), 256, 0, ctx->stream>>>(ctx->fb.ptr, ctx->rb_rgb[slot].ptr,
                                                                                      npix);
        VXA_CUDA(cudaGetLastError());
    }
    VXA_CUDA(cudaEventRecord(ctx->rb_packed[slot], ctx->stream));
    // the previous frame's D2H goes to the copy engine now, behind this frame's upload
    if (int rc = flush_readback(ctx); rc != VXA_OK) return rc;
    ctx->rb_pending = true;
    ctx->rb_pending_slot = slot;
    ctx->rb_pending_out = rgb_out;
    ctx->rb_pending_bytes = npix * 3;
    ctx->d2h += npix * 3;
    *ticket = ctx->rb_next++;
    return VXA_OK;
}

int vxa_wait_readback(vxa_ctx* ctx, uint64_t ticket) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (ticket >= ctx->rb_next) return fail(VXA_ERR_INVALID, "unknown readback ticket");
    if (ticket + 1 == ctx->rb_next)
        if (int rc = flush_readback(ctx); rc != VXA_OK) return rc;
    // the slot's event marks this ticket's D2H or a later one on the same FIFO
    // copy stream, so waiting for it covers this ticket
    VXA_CUDA(cudaEventSynchronize(ctx->rb_done[ticket & 1u]));
    return VXA_OK;
}

int vxa_synchronize(vxa_ctx* ctx) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (int rc = flush_readback(ctx); rc != VXA_OK) return rc; // streamed images land too
    VXA_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->copy_stream) VXA_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    return VXA_OK;
}

int vxa_stats_read(vxa_ctx* ctx, vxa_stats* stats) {
    if (ctx == nullptr || stats == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    *stats = vxa_stats{};
    return read_counters(ctx, stats);
}

int vxa_stats_reset(vxa_ctx* ctx) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    VXA_CUDA(cudaMemsetAsync(ctx->counters.ptr, 0, 8 * sizeof(unsigned long long), ctx->stream));
    ctx->k_count = 0;
    ctx->aux_launches = 0;
    ctx->h2d = ctx->d2h = 0;
    ctx->n_rays = ctx->n_sphere_tests = 0;
    return VXA_OK;
}

int vxa_read_framebuffer(vxa_ctx* ctx, uint8_t* rgb_out, int32_t width, int32_t height) {
    if (ctx == nullptr || rgb_out == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (width != ctx->fb_w || height != ctx->fb_h) return fail(VXA_ERR_INVALID, "framebuffer size mismatch");
    const size_t npix = static_cast<size_t>(width) * height;
    VXA_CUDA(ctx->rgb.ensure(npix * 3 + 16));
    const size_t quads = (npix + 3) / 4;
    pack_rgb<<<static_cast<unsigned>((quads + 255) / 256), 256, 0, ctx->stream>>>(ctx->fb.ptr, ctx->rgb.ptr, npix);
    VXA_CUDA(cudaGetLastError());
    VXA_CUDA(cudaMemcpyAsync(rgb_out, ctx->rgb.ptr, npix * 3, cudaMemcpyDeviceToHost, ctx->stream));
    VXA_CUDA(cudaStreamSynchronize(ctx->stream));
    return VXA_OK;
}

int vxa_host_register(vxa_ctx* ctx, void* ptr, size_t bytes) {
    if (ctx == nullptr || ptr == nullptr || bytes == 0) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    VXA_CUDA(cudaSetDevice(ctx->device));
    VXA_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
    return VXA_OK;
}

int vxa_host_unregister(vxa_ctx* ctx, void* ptr) {
    if (ctx == nullptr || ptr == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    VXA_CUDA(cudaSetDevice(ctx->device));
    VXA_CUDA(cudaHostUnregister(ptr));
    return VXA_OK;
}

int vxa_timer_begin(vxa_ctx* ctx) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    VXA_CUDA(cudaEventRecord(ctx->t_a, ctx->stream));
    return VXA_OK;
}

int vxa_timer_end(vxa_ctx* ctx, double* elapsed_ms) {
    if (ctx == nullptr || elapsed_ms == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    VXA_CUDA(cudaEventRecord(ctx->t_b, ctx->stream));
    VXA_CUDA(cudaEventSynchronize(ctx->t_b));
    float ms = 0.f;
    VXA_CUDA(cudaEventElapsedTime(&ms, ctx->t_a, ctx->t_b));
    *elapsed_ms = ms;
    return VXA_OK;
}

namespace {
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__global__ void delay_kernel(uint32_t ns) {
    const unsigned long long t0 = globaltimer_ns();
    while (globaltimer_ns() - t0 < ns) __nanosleep(1000);
}
} // namespace

int vxa_stream_delay(vxa_ctx* ctx, uint32_t microseconds) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    VXA_CUDA(cudaSetDevice(ctx->device));
    delay_kernel<<<1, 1, 0, ctx->stream>>>(1000u * std::min<uint32_t>(microseconds, 1000000u));
    VXA_CUDA(cudaGetLastError());
    return VXA_OK;
}

int vxa_flush_l2(vxa_ctx* ctx) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    const size_t bytes = size_t{256} << 20; // 2x the 126 MB L2
    VXA_CUDA(ctx->l2_scratch.ensure(bytes));
    VXA_CUDA(cudaMemsetAsync(ctx->l2_scratch.ptr, ctx->inst_slot, bytes, ctx->stream));
    return VXA_OK;
}

void* vxa_stream(vxa_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int vxa_fb_export(vxa_ctx* ctx, int32_t width, int32_t height, void* ipc_handle_out) {
    if (ctx == nullptr || ipc_handle_out == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (width < 1 || height < 1) return fail(VXA_ERR_INVALID, "bad framebuffer size");
    VXA_CUDA(cudaSetDevice(ctx->device));
    VXA_CUDA(ctx->fb.ensure(static_cast<size_t>(width) * height));
    ctx->fb_w = width;
    ctx->fb_h = height;
    cudaIpcMemHandle_t h;
    VXA_CUDA(cudaIpcGetMemHandle(&h, ctx->fb.ptr));
    std::memcpy(ipc_handle_out, &h, sizeof(h));
    return VXA_OK;
}

int vxa_fb_import(vxa_ctx* ctx, int32_t width, int32_t height, const void* ipc_handle) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    VXA_CUDA(cudaSetDevice(ctx->device));
    if (ctx->peer_fb) {
        cudaIpcCloseMemHandle(ctx->peer_fb);
        ctx->peer_fb = nullptr;
    }
    if (ipc_handle == nullptr) return VXA_OK; // detach: frames store into the local framebuffer again
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, sizeof(h));
    void* p = nullptr;
    VXA_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->peer_fb = static_cast<uint32_t*>(p);
    ctx->peer_w = width;
    ctx->peer_h = height;
    return VXA_OK;
}

namespace {
// ---- frame completion flags (vxa_frame_open / vxa_frame_close) -------------
// One thread each. The store is a system-scope release after a full fence, so
// every write this device made before it (the frame kernel's peer stores into
// rank 0's framebuffer, themselves fenced at system scope by their threads)
// is visible to a thread that acquires the flag. The wait spins with
// system-scope acquire loads (the flags are written over NVLink) and gives up
// after timeout_ns, latching err: a lost rank never hangs the device.
__global__ void sync_store_kernel(unsigned int* flag, unsigned int v) {
    asm volatile("fence.sc.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned int load_acquire_sys(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// flags[0 .. n) must all reach v (frame numbers increase by one per frame;
// the difference is compared as a signed value, so wrap-around is harmless).
__global__ void sync_wait_kernel(const unsigned int* flags, int n, unsigned int v, unsigned long long timeout_ns,
                                 unsigned int* err) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < n; ++i) {
        unsigned int ns = 32;
        while (static_cast<int>(load_acquire_sys(flags + i) - v) < 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) {
                atomicOr(err, 1u);
                return;
            }
            __nanosleep(ns);
            ns = ns < 1024 ? 2 * ns : ns;
        }
    }
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// VXA_SYNC_HOST: poll flags[0 .. n) from the host until all reach v.
int host_poll(vxa_ctx* ctx, const unsigned int* flags, int n, unsigned int v) {
    const auto t0 = std::chrono::steady_clock::now();
    while (true) {
        VXA_CUDA(cudaMemcpyAsync(ctx->sync_host, flags, sizeof(unsigned int) * n, cudaMemcpyDeviceToHost,
                                 ctx->poll_stream));
        VXA_CUDA(cudaStreamSynchronize(ctx->poll_stream));
        bool all = true;
        for (int i = 0; i < n && all; ++i) all = static_cast<int>(ctx->sync_host[i] - v) >= 0;
        if (all) return VXA_OK;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms * 1e6 > static_cast<double>(ctx->sync_timeout_ns))
            return fail(VXA_ERR_CUDA, "vxa_frame sync: timed out waiting for another rank");
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

int sync_common(vxa_ctx* ctx, int32_t rank, int32_t world) {
    if (world < 2 || world > vxa_ctx::kSyncRanks || rank < 0 || rank >= world)
        return fail(VXA_ERR_INVALID, "sync: rank/world out of range");
    VXA_CUDA(cudaSetDevice(ctx->device));
    VXA_CUDA(ctx->sync_err.ensure(1));
    VXA_CUDA(cudaMemset(ctx->sync_err.ptr, 0, sizeof(unsigned int)));
    if (ctx->poll_stream == nullptr) VXA_CUDA(cudaStreamCreateWithFlags(&ctx->poll_stream, cudaStreamNonBlocking));
    if (ctx->sync_host == nullptr)
        VXA_CUDA(cudaMallocHost(&ctx->sync_host, sizeof(unsigned int) * (vxa_ctx::kSyncRanks + 2)));
    ctx->sync_rank = rank;
    ctx->sync_world = world;
    ctx->sync_seq = 0;
    return VXA_OK;
}
} // namespace

int vxa_sync_export(vxa_ctx* ctx, int32_t world, void* ipc_handle_out) {
    if (ctx == nullptr || ipc_handle_out == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (int rc = sync_common(ctx, 0, world); rc != VXA_OK) return rc;
    VXA_CUDA(ctx->sync_own.ensure(vxa_ctx::kSyncRanks + 2));
    VXA_CUDA(cudaMemset(ctx->sync_own.ptr, 0, sizeof(unsigned int) * (vxa_ctx::kSyncRanks + 2)));
    cudaIpcMemHandle_t h;
    VXA_CUDA(cudaIpcGetMemHandle(&h, ctx->sync_own.ptr));
    std::memcpy(ipc_handle_out, &h, sizeof(h));
    ctx->sync_flags = ctx->sync_own.ptr;
    return VXA_OK;
}

int vxa_sync_import(vxa_ctx* ctx, int32_t rank, int32_t world, const void* ipc_handle) {
    if (ctx == nullptr || ipc_handle == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (rank == 0) return fail(VXA_ERR_INVALID, "sync: rank 0 exports the flag block");
    if (int rc = sync_common(ctx, rank, world); rc != VXA_OK) return rc;
    if (ctx->sync_peer) {
        cudaIpcCloseMemHandle(ctx->sync_peer);
        ctx->sync_peer = nullptr;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, sizeof(h));
    void* p = nullptr;
    VXA_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->sync_peer = static_cast<unsigned int*>(p);
    ctx->sync_flags = ctx->sync_peer;
    return VXA_OK;
}

int vxa_sync_configure(vxa_ctx* ctx, int32_t mode, uint32_t timeout_ms) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (mode != VXA_SYNC_DEVICE && mode != VXA_SYNC_HOST) return fail(VXA_ERR_INVALID, "sync: unknown mode");
    ctx->sync_mode = mode;
    if (timeout_ms > 0) ctx->sync_timeout_ns = static_cast<uint64_t>(timeout_ms) * 1000000ull;
    return VXA_OK;
}

int vxa_frame_open(vxa_ctx* ctx) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (ctx->sync_flags == nullptr) return fail(VXA_ERR_INVALID, "sync: no flag block (vxa_sync_export/import)");
    VXA_CUDA(cudaSetDevice(ctx->device));
    const unsigned int v = ++ctx->sync_seq;
    if (ctx->sync_rank == 0) {
        sync_store_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sync_flags, v);
        ++ctx->aux_launches;
    } else if (ctx->sync_mode == VXA_SYNC_DEVICE) {
        sync_wait_kernel<<<1, 1, 0, ctx->stream>>>(ctx->sync_flags, 1, v, ctx->sync_timeout_ns, ctx->sync_err.ptr);
        ++ctx->aux_launches;
    } else {
        if (int rc = host_poll(ctx, ctx->sync_flags, 1, v); rc != VXA_OK) return rc;
    }
    VXA_CUDA(cudaGetLastError());
    return VXA_OK;
}

int vxa_frame_close(vxa_ctx* ctx) {
    if (ctx == nullptr) return fail(VXA_ERR_INVALID, "null context");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (ctx->sync_flags == nullptr) return fail(VXA_ERR_INVALID, "sync: no flag block (vxa_sync_export/import)");
    VXA_CUDA(cudaSetDevice(ctx->device));
    const unsigned int v = ctx->sync_seq;
    unsigned int* done = ctx->sync_flags + 2; // done[r] at word 2 + r
    if (ctx->sync_rank != 0) {
        sync_store_kernel<<<1, 1, 0, ctx->stream>>>(done + ctx->sync_rank, v);
        ++ctx->aux_launches;
    } else if (ctx->sync_mode == VXA_SYNC_DEVICE) {
        sync_wait_kernel<<<1, 1, 0, ctx->stream>>>(done + 1, ctx->sync_world - 1, v, ctx->sync_timeout_ns,
                                                   ctx->sync_err.ptr);
        ++ctx->aux_launches;
    } else {
        if (int rc = host_poll(ctx, done + 1, ctx->sync_world - 1, v); rc != VXA_OK) return rc;
    }
    VXA_CUDA(cudaGetLastError());
    return VXA_OK;
}

int vxa_sync_status(vxa_ctx* ctx, int32_t* timed_out) {
    if (ctx == nullptr || timed_out == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    *timed_out = 0;
    if (ctx->sync_err.ptr == nullptr) return VXA_OK;
    unsigned int e = 0;
    VXA_CUDA(cudaStreamSynchronize(ctx->stream));
    VXA_CUDA(cudaMemcpy(&e, ctx->sync_err.ptr, sizeof(e), cudaMemcpyDeviceToHost));
    *timed_out = e ? 1 : 0;
    return VXA_OK;
}

int vxa_framebuffer_readback(vxa_ctx* ctx, int32_t width, int32_t height, uint8_t* rgb_out, uint64_t* ticket) {
    if (ctx == nullptr || rgb_out == nullptr || ticket == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (width != ctx->fb_w || height != ctx->fb_h || ctx->fb.ptr == nullptr)
        return fail(VXA_ERR_INVALID, "framebuffer size mismatch");
    VXA_CUDA(cudaSetDevice(ctx->device));
    const size_t npix = static_cast<size_t>(width) * height;
    const int slot = static_cast<int>(ctx->rb_next & 1u);
    VXA_CUDA(ctx->rb_rgb[slot].ensure(npix * 3 + 16));
    VXA_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->rb_done[slot], 0)); // the slot's previous D2H
    const size_t quads = (npix + 3) / 4;
    pack_rgb<<<static_cast<unsigned>((quads + 255) / 256), 256, 0, ctx->stream>>>(ctx->fb.ptr, ctx->rb_rgb[slot].ptr,
                                                                                  npix);
    VXA_CUDA(cudaGetLastError());
    ++ctx->aux_launches;
    VXA_CUDA(cudaEventRecord(ctx->rb_packed[slot], ctx->stream));
    if (int rc = flush_readback(ctx); rc != VXA_OK) return rc;
    ctx->rb_pending = true;
    ctx->rb_pending_slot = slot;
    ctx->rb_pending_out = rgb_out;
    ctx->rb_pending_bytes = npix * 3;
    ctx->d2h += npix * 3;
    *ticket = ctx->rb_next++;
    return VXA_OK;
}

int32_t vxa_tile_owner(int32_t x, int32_t y, int32_t width, int32_t height, int32_t world) {
    if (world < 1 || x < 0 || y < 0 || x >= width || y >= height) return -1;
    return tile_owner(x, y, width, world);
}

namespace {
// One thread per pixel of the rank's tiles: tile k is super-tile s = k * world + rank.
__global__ void tiles_copy(uint32_t* fb, uint32_t* buf, int32_t width, int32_t height, uint32_t n_super_x,
                           int32_t rank, int32_t world, uint32_t tiles, bool pack) {
    const uint64_t i = blockIdx.x * uint64_t{blockDim.x} + threadIdx.x;
    if (i >= uint64_t{tiles} * kSuper * kSuper) return;
    const uint32_t k = static_cast<uint32_t>(i / (kSuper * kSuper)), p = static_cast<uint32_t>(i % (kSuper * kSuper));
    const uint32_t s = k * static_cast<uint32_t>(world) + static_cast<uint32_t>(rank);
    const int32_t x = static_cast<int32_t>((s % n_super_x) * kSuper + p % kSuper);
    const int32_t y = static_cast<int32_t>((s / n_super_x) * kSuper + p / kSuper);
    if (x >= width || y >= height) {
        if (pack) buf[i] = 0u; // padding of an edge tile
        return;
    }
    const size_t f = static_cast<size_t>(y) * width + x;
    if (pack)
        buf[i] = fb[f];
    else
        fb[f] = buf[i];
}

uint32_t tiles_of(int32_t width, int32_t height, int32_t rank, int32_t world) {
    const uint32_t n_super = super_tiles_x(width) * static_cast<uint32_t>((height + kSuper - 1) / kSuper);
    return (n_super + static_cast<uint32_t>(world - rank) - 1) / static_cast<uint32_t>(world);
}

int tiles_move(vxa_ctx* ctx, int32_t width, int32_t height, int32_t rank, int32_t world, void* buf, bool pack) {
    if (ctx == nullptr || buf == nullptr) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    if (width < 1 || height < 1 || world < 1 || rank < 0 || rank >= world)
        return fail(VXA_ERR_INVALID, "bad frame size or partition");
    if (ctx->fb_w != width || ctx->fb_h != height) return fail(VXA_ERR_INVALID, "framebuffer size mismatch");
    const uint32_t tiles = tiles_of(width, height, rank, world);
    const uint64_t n = uint64_t{tiles} * kSuper * kSuper;
    if (n == 0) return VXA_OK;
    VXA_CUDA(cudaSetDevice(ctx->device));
    tiles_copy<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->fb.ptr, static_cast<uint32_t*>(buf), width, height, super_tiles_x(width), rank, world, tiles, pack);
    VXA_CUDA(cudaGetLastError());
    return VXA_OK;
}
} // namespace

int vxa_tiles_count(int32_t width, int32_t height, int32_t rank, int32_t world, uint32_t* count) {
    if (count == nullptr || width < 1 || height < 1 || world < 1 || rank < 0 || rank >= world)
        return fail(VXA_ERR_INVALID, "bad frame size or partition");
    *count = tiles_of(width, height, rank, world);
    return VXA_OK;
}

int vxa_tiles_pack(vxa_ctx* ctx, int32_t width, int32_t height, int32_t rank, int32_t world, void* dst_device) {
    return tiles_move(ctx, width, height, rank, world, dst_device, true);
}

int vxa_tiles_unpack(vxa_ctx* ctx, int32_t width, int32_t height, int32_t rank, int32_t world, const void* src_device) {
    return tiles_move(ctx, width, height, rank, world, const_cast<void*>(src_device), false);
}

int vxa_traverse(vxa_ctx* ctx, uint32_t model, const vxa_local_ray* rays, uint32_t n, uint32_t precision,
                 vxa_traverse_hit* hits, vxa_visit* log, uint32_t log_capacity) {
    static_assert(sizeof(vxa_local_ray) == sizeof(TraverseRayIn));
    static_assert(sizeof(vxa_traverse_hit) == sizeof(TraverseRayOut));
    static_assert(sizeof(vxa_visit) == sizeof(VisitOut));
    if (ctx == nullptr || (n > 0 && (rays == nullptr || hits == nullptr))) return fail(VXA_ERR_INVALID, "null argument");
    std::lock_guard<std::recursive_mutex> lock_(ctx->mu);
    const auto it = ctx->models.find(model);
    if (it == ctx->models.end()) return fail(VXA_ERR_INVALID, "unknown model handle");
    if (n == 0) return VXA_OK;
    VXA_CUDA(cudaSetDevice(ctx->device));
    VXA_CUDA(ctx->rays.ensure(n));
    VXA_CUDA(ctx->hits.ensure(n));
    VisitOut* dlog = nullptr;
    if (log != nullptr && log_capacity > 0) {
        VXA_CUDA(ctx->visits.ensure(size_t{n} * log_capacity));
        dlog = ctx->visits.ptr;
    }
    VXA_CUDA(cudaMemcpyAsync(ctx->rays.ptr, rays, sizeof(TraverseRayIn) * n, cudaMemcpyHostToDevice, ctx->stream));
    const cudaError_t e = precision == VXA_FP64
                              ? launch_traverse_f64(it->second.dev, ctx->rays.ptr, n, ctx->hits.ptr, dlog,
                                                    dlog ? log_capacity : 0, ctx->stream)
                              : launch_traverse_f32(it->second.dev, ctx->rays.ptr, n, ctx->hits.ptr, dlog,
                                                    dlog ? log_capacity : 0, ctx->stream);
    if (e != cudaSuccess) return fail(VXA_ERR_CUDA, std::string("traverse launch: ") + cudaGetErrorString(e));
    VXA_CUDA(cudaMemcpyAsync(hits, ctx->hits.ptr, sizeof(TraverseRayOut) * n, cudaMemcpyDeviceToHost, ctx->stream));
    if (dlog)
        VXA_CUDA(cudaMemcpyAsync(log, dlog, sizeof(VisitOut) * n * size_t{log_capacity}, cudaMemcpyDeviceToHost,
                                 ctx->stream));
    VXA_CUDA(cudaStreamSynchronize(ctx->stream));
    return VXA_OK;
}

} // extern "C"
