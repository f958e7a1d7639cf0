// Host side of the drop-in boundary: the process-wide vxa context, the device
// model cache and status -> exception translation.
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>
#include <string>

#include "voxanim/gpu.hpp"

namespace voxanim::gpu {

namespace {

std::mutex g_mu;
vxa_ctx* g_ctx = nullptr;
int g_precision = -1; // -1: read VOXANIM_PRECISION on first use

struct CachedModel {
    const void* nodes;
    const void* attrs;
    std::size_t node_count, attr_count;
    std::uint32_t depth;
    std::uint64_t signature;
    std::uint32_t handle;
    std::uint64_t bytes;
};

std::list<CachedModel> g_cache; // most recently used first
std::uint64_t g_cache_bytes = 0;

std::uint64_t mix64(std::uint64_t h, std::uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
}

std::uint64_t fold_bytes(std::uint64_t h, const void* p, std::size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    std::size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        std::uint64_t w;
        std::memcpy(&w, b + i, 8);
        h = mix64(h, w);
    }
    for (; i < n; ++i) h = mix64(h, b[i]);
    return h;
}

// Whole content for tiny models, a strided sample otherwise: it tells apart
// different models that reuse one storage address (models are shared
// immutably, shared_ptr<const SvoModel>), and it runs on every frame, so it
// stays small (a full hash of a 1 MB model per call would dominate small frames).
std::uint64_t signature(const SvoModel& m) {
    std::uint64_t h = mix64(m.depth, m.nodes.size() * 1315423911ull + m.attributes.size());
    const std::size_t nb = m.nodes.size() * sizeof(SvoNode), ab = m.attributes.size() * sizeof(VoxelAttribute);
    if (nb + ab <= 4096) {
        h = fold_bytes(h, m.nodes.data(), nb);
        return fold_bytes(h, m.attributes.data(), ab);
    }
    const std::size_t nn = m.nodes.size(), na = m.attributes.size();
    for (std::size_t k = 0; k < 64; ++k) {
        h = fold_bytes(h, &m.nodes[(k * 2654435761ull) % nn], sizeof(SvoNode));
        if (na) h = fold_bytes(h, &m.attributes[(k * 40503ull) % na], sizeof(VoxelAttribute));
    }
    return h;
}

std::uint64_t cache_budget() {
    const char* env = std::getenv("VOXANIM_MODEL_CACHE_MB");
    return (env ? std::strtoull(env, nullptr, 10) : 16384ull) << 20;
}

vxa_ctx* ctx_locked() {
    if (g_ctx == nullptr) check(vxa_create(-1, &g_ctx), "vxa_create");
    return g_ctx;
}

} // namespace

void check(int status, const char* what) {
    if (status == VXA_OK) return;
    const std::string msg = std::string(what) + ": " + vxa_last_error();
    if (status == VXA_ERR_INVALID || status == VXA_ERR_MODEL) throw ValidationError(msg);
    throw DeviceError(msg);
}

vxa_ctx* context() {
    std::lock_guard<std::mutex> lk(g_mu);
    return ctx_locked();
}

Precision default_precision() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_precision < 0) {
        const char* env = std::getenv("VOXANIM_PRECISION");
        g_precision = (env && std::strcmp(env, "fp64") == 0) ? VXA_FP64 : VXA_FP32;
    }
    return static_cast<Precision>(g_precision);
}

void set_default_precision(Precision p) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_precision = static_cast<int>(p);
}

std::uint32_t model_handle(const SvoModel& m) {
    std::lock_guard<std::mutex> lk(g_mu);
    vxa_ctx* ctx = ctx_locked();
    const std::uint64_t sig = signature(m);
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        if (it->nodes == m.nodes.data() && it->attrs == m.attributes.data() && it->node_count == m.nodes.size() &&
            it->attr_count == m.attributes.size() && it->depth == m.depth && it->signature == sig) {
            g_cache.splice(g_cache.begin(), g_cache, it);
            return g_cache.front().handle;
        }
    }
    std::uint32_t handle = 0;
    check(vxa_upload_model(ctx, m.nodes.data(), static_cast<std::uint32_t>(m.nodes.size()), m.attributes.data(),
                           static_cast<std::uint32_t>(m.attributes.size()), m.depth, &handle),
          "vxa_upload_model");
    std::uint64_t bytes = 0;
    vxa_model_info(ctx, handle, &bytes, nullptr);
    g_cache.push_front({m.nodes.data(), m.attributes.data(), m.nodes.size(), m.attributes.size(), m.depth, sig, handle,
                        bytes});
    g_cache_bytes += bytes;
    // Evict least recently used models beyond the budget (never the new one).
    const std::uint64_t budget = cache_budget();
    while (g_cache_bytes > budget && g_cache.size() > 1) {
        const CachedModel& victim = g_cache.back();
        vxa_release_model(ctx, victim.handle);
        g_cache_bytes -= victim.bytes;
        g_cache.pop_back();
    }
    return handle;
}

SvoModel build_from_grid(const VoxelGrid& grid, std::uint32_t depth) {
    // the reference's argument checks (svo.cpp:80-87), same messages
    if (depth < 1 || depth > 16)
        throw ValidationError("octree depth must be in [1, 16], got " + std::to_string(depth));
    if (grid.resolution() != (1u << depth))
        throw ValidationError("grid resolution " + std::to_string(grid.resolution()) +
                              " does not match 2^depth = " + std::to_string(1u << depth));
    const ColorSpec& cs = grid.colors();
    const std::uint32_t rgba = cs.constant.r | (std::uint32_t{cs.constant.g} << 8) |
                               (std::uint32_t{cs.constant.b} << 16) | (std::uint32_t{cs.constant.a} << 24);
    std::lock_guard<std::mutex> lk(g_mu);
    vxa_ctx* ctx = ctx_locked();
    std::uint32_t handle = 0;
    std::uint64_t nn = 0, na = 0;
    check(vxa_build_model(ctx, grid.words(), depth, static_cast<std::uint32_t>(cs.mode), rgba, &handle, &nn, &na),
          "vxa_build_model");
    SvoModel m;
    m.depth = depth;
    try {
        m.nodes.resize(nn);
        m.attributes.resize(na);
        check(vxa_model_download(ctx, handle, m.nodes.data(), nn, reinterpret_cast<std::uint32_t*>(m.attributes.data()),
                                 na),
              "vxa_model_download");
    } catch (...) {
        vxa_release_model(ctx, handle);
        throw;
    }
    std::uint64_t bytes = 0;
    vxa_model_info(ctx, handle, &bytes, nullptr);
    g_cache.push_front({m.nodes.data(), m.attributes.data(), m.nodes.size(), m.attributes.size(), m.depth, signature(m),
                        handle, bytes});
    g_cache_bytes += bytes;
    return m;
}

} // namespace voxanim::gpu
