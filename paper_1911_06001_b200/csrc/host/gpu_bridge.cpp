// Host side of the drop-in boundary: the process-wide vxa context, the device
// model cache and status -> exception translation.
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <list>
#include <memory>
#include <mutex>
#include <string>

#include "voxanim/gpu.hpp"

namespace voxanim::gpu {

namespace {

std::mutex g_mu;
vxa_ctx* g_ctx = nullptr;
int g_precision = -1; // -1: read VOXANIM_PRECISION on first use

struct CachedModel {
    // Scene models (shared_ptr<const SvoModel>, scene.hpp:20): keyed by the
    // owner's control block, which this weak_ptr keeps allocated, so a later
    // model can never reuse the key; the entry is released once the model is
    // gone. Raw references (traverse API) use the storage key below only.
    std::weak_ptr<const SvoModel> owner;
    bool owned;
    std::uint64_t frame; // frame generation that last used the handle (never evicted within it)
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
std::uint64_t g_frame = 1; // current frame generation (begin_model_frame)

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

namespace {

bool same_storage(const CachedModel& c, const SvoModel& m, std::uint64_t sig) {
    return c.nodes == m.nodes.data() && c.attrs == m.attributes.data() && c.node_count == m.nodes.size() &&
           c.attr_count == m.attributes.size() && c.depth == m.depth && c.signature == sig;
}

// Releases the device copies of scene models that no longer exist.
void purge_expired(vxa_ctx* ctx) {
    for (auto it = g_cache.begin(); it != g_cache.end();) {
        if (it->owned && it->owner.expired()) {
            vxa_release_model(ctx, it->handle);
            g_cache_bytes -= it->bytes;
            it = g_cache.erase(it);
        } else {
            ++it;
        }
    }
}

std::uint32_t upload_locked(vxa_ctx* ctx, const SvoModel& m, std::uint64_t sig,
                            const std::shared_ptr<const SvoModel>* owner) {
    std::uint32_t handle = 0;
    check(vxa_upload_model(ctx, m.nodes.data(), static_cast<std::uint32_t>(m.nodes.size()), m.attributes.data(),
                           static_cast<std::uint32_t>(m.attributes.size()), m.depth, &handle),
          "vxa_upload_model");
    std::uint64_t bytes = 0;
    vxa_model_info(ctx, handle, &bytes, nullptr);
    g_cache.push_front({owner ? std::weak_ptr<const SvoModel>(*owner) : std::weak_ptr<const SvoModel>(), owner != nullptr,
                        g_frame, m.nodes.data(), m.attributes.data(), m.nodes.size(), m.attributes.size(), m.depth, sig,
                        handle, bytes});
    g_cache_bytes += bytes;
    // Evict least recently used models beyond the budget: never the new one, nor
    // one a frame being assembled already holds (same generation).
    const std::uint64_t budget = cache_budget();
    for (auto it = std::prev(g_cache.end()); g_cache_bytes > budget && it != g_cache.begin();) {
        auto victim = it--;
        if (victim->frame == g_frame) continue;
        vxa_release_model(ctx, victim->handle);
        g_cache_bytes -= victim->bytes;
        g_cache.erase(victim);
    }
    return handle;
}

} // namespace

std::uint64_t begin_model_frame() {
    std::lock_guard<std::mutex> lk(g_mu);
    return ++g_frame;
}

std::uint32_t model_handle(const std::shared_ptr<const SvoModel>& model) {
    if (!model) throw ValidationError("null model");
    std::lock_guard<std::mutex> lk(g_mu);
    vxa_ctx* ctx = ctx_locked();
    purge_expired(ctx);
    const SvoModel& m = *model;
    const std::uint64_t sig = signature(m);
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        if (!it->owned || it->owner.owner_before(model) || model.owner_before(it->owner)) continue;
        if (same_storage(*it, m, sig)) {
            it->frame = g_frame;
            g_cache.splice(g_cache.begin(), g_cache, it);
            return g_cache.front().handle;
        }
        // the same owner with different contents (edited in place): re-upload
        vxa_release_model(ctx, it->handle);
        g_cache_bytes -= it->bytes;
        g_cache.erase(it);
        break;
    }
    // a device copy made for the same storage before the model was shared (e.g.
    // build_from_grid's, or a traverse call's) is adopted by its owner
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        if (!it->owned && same_storage(*it, m, sig)) {
            it->owner = model;
            it->owned = true;
            it->frame = g_frame;
            g_cache.splice(g_cache.begin(), g_cache, it);
            return g_cache.front().handle;
        }
    }
    return upload_locked(ctx, m, sig, &model);
}

std::uint32_t model_handle(const SvoModel& m) {
    std::lock_guard<std::mutex> lk(g_mu);
    vxa_ctx* ctx = ctx_locked();
    purge_expired(ctx);
    const std::uint64_t sig = signature(m);
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        if (!it->owned && same_storage(*it, m, sig)) {
            it->frame = g_frame;
            g_cache.splice(g_cache.begin(), g_cache, it);
            return g_cache.front().handle;
        }
    }
    return upload_locked(ctx, m, sig, nullptr);
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
    g_cache.push_front({std::weak_ptr<const SvoModel>(), false, g_frame, m.nodes.data(), m.attributes.data(),
                        m.nodes.size(), m.attributes.size(), m.depth, signature(m), handle, bytes});
    g_cache_bytes += bytes;
    return m;
}

} // namespace voxanim::gpu
