// Flat C binding of the voxanim C++ API (include/voxanim_capi.h).
#include "voxanim_capi.h"

#include <chrono>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "bench_scenes.hpp"
#include "voxanim/gpu.hpp"
#include "voxanim/ingest.hpp"
#include "voxanim/procedural.hpp"
#include "voxanim/renderer.hpp"
#include "voxanim/svo.hpp"

struct vxn_model {
    std::shared_ptr<const voxanim::SvoModel> m;
};
struct vxn_scene {
    voxanim::Scene s;
};
struct vxn_hbo {
    voxanim::HitBuffer b;
};

namespace {

thread_local std::string g_err;

template <class F> auto guard(F&& f, decltype(f()) on_error) -> decltype(f()) {
    try {
        return f();
    } catch (const std::exception& e) {
        g_err = e.what();
    } catch (...) {
        g_err = "unknown C++ exception";
    }
    return on_error;
}

vxn_model* wrap(voxanim::SvoModel&& m) {
    return new vxn_model{std::make_shared<const voxanim::SvoModel>(std::move(m))};
}

} // namespace

extern "C" {

const char* vxn_last_error(void) { return g_err.c_str(); }

vxn_model* vxn_model_procedural(int shell, uint32_t depth) {
    return guard(
        [&] {
            return wrap(voxanim::build_procedural(
                shell ? voxanim::ProceduralShape::ShellSphere : voxanim::ProceduralShape::SolidSphere, depth));
        },
        static_cast<vxn_model*>(nullptr));
}

vxn_model* vxn_model_dense_sphere(uint32_t depth) {
    return guard(
        [&] {
            return wrap(voxanim::build_from_grid(voxanim::gen_primitive(voxanim::PrimitiveKind::Sphere, depth), depth));
        },
        static_cast<vxn_model*>(nullptr));
}

vxn_model* vxn_model_random(uint64_t seed, uint32_t depth, double fill) {
    return guard(
        [&] {
            std::mt19937_64 rng(seed);
            voxanim::VoxelGrid g(1u << depth);
            std::uniform_real_distribution<double> coin(0.0, 1.0);
            const std::uint32_t n = g.resolution();
            for (std::uint32_t x = 0; x < n; ++x)
                for (std::uint32_t y = 0; y < n; ++y)
                    for (std::uint32_t z = 0; z < n; ++z)
                        if (coin(rng) < fill) g.set(x, y, z);
            return wrap(voxanim::build_from_grid(g, depth));
        },
        static_cast<vxn_model*>(nullptr));
}

vxn_model* vxn_model_full_cube(void) {
    return guard(
        [&] {
            voxanim::VoxelGrid g(2);
            for (std::uint32_t i = 0; i < 8; ++i) g.set(i >> 2, (i >> 1) & 1u, i & 1u);
            return wrap(voxanim::build_from_grid(g, 1));
        },
        static_cast<vxn_model*>(nullptr));
}

vxn_model* vxn_model_from_grid(const uint64_t* words, uint32_t depth, uint32_t color_mode, uint32_t color_rgba,
                               int device) {
    return guard(
        [&] {
            if (words == nullptr || depth < 1 || depth > 10 || color_mode > 2)
                throw voxanim::ValidationError("vxn_model_from_grid: bad arguments");
            voxanim::ColorSpec cs;
            cs.mode = static_cast<voxanim::ColorMode>(color_mode);
            cs.constant = {static_cast<std::uint8_t>(color_rgba), static_cast<std::uint8_t>(color_rgba >> 8),
                           static_cast<std::uint8_t>(color_rgba >> 16), static_cast<std::uint8_t>(color_rgba >> 24)};
            voxanim::VoxelGrid g(1u << depth, cs);
            g.assign_words(words);
            return wrap(device ? voxanim::gpu::build_from_grid(g, depth) : voxanim::build_from_grid(g, depth));
        },
        static_cast<vxn_model*>(nullptr));
}

int64_t vxn_grid_primitive(int kind, uint32_t depth, uint64_t* out, size_t cap_words, uint32_t* grid_depth) {
    return guard(
        [&]() -> int64_t {
            if (kind < 0 || kind > 3) throw voxanim::ValidationError("unknown primitive kind");
            const voxanim::VoxelGrid g = voxanim::gen_primitive(static_cast<voxanim::PrimitiveKind>(kind), depth);
            if (grid_depth) *grid_depth = g.depth();
            if (out == nullptr) return static_cast<int64_t>(g.word_count());
            if (cap_words < g.word_count()) throw voxanim::ValidationError("output too small");
            std::memcpy(out, g.words(), 8 * g.word_count());
            return static_cast<int64_t>(g.word_count());
        },
        int64_t{-1});
}

int vxn_model_save(const vxn_model* m, const char* path) {
    return guard(
        [&] {
            voxanim::save_svo(path, *m->m);
            return 0;
        },
        -1);
}

vxn_scene* vxn_scene_load(const char* path, int width, int height) {
    return guard(
        [&] {
            auto* s = new vxn_scene{voxanim::load_scene_file(path)};
            s->s.camera.width = width;
            s->s.camera.height = height;
            return s;
        },
        static_cast<vxn_scene*>(nullptr));
}

vxn_model* vxn_model_deserialize(const uint8_t* bytes, size_t n) {
    return guard([&] { return wrap(voxanim::deserialize(std::span<const std::uint8_t>(bytes, n))); },
                 static_cast<vxn_model*>(nullptr));
}

int64_t vxn_model_serialize(const vxn_model* m, uint8_t* out, size_t cap) {
    return guard(
        [&]() -> int64_t {
            const auto bytes = voxanim::serialize(*m->m);
            if (out != nullptr) {
                if (cap < bytes.size()) throw voxanim::ValidationError("serialize: buffer too small");
                std::memcpy(out, bytes.data(), bytes.size());
            }
            return static_cast<int64_t>(bytes.size());
        },
        int64_t{-1});
}

int vxn_model_info(const vxn_model* m, uint32_t* depth, uint64_t* nodes, uint64_t* attrs) {
    if (m == nullptr) return -1;
    if (depth) *depth = m->m->depth;
    if (nodes) *nodes = m->m->nodes.size();
    if (attrs) *attrs = m->m->attributes.size();
    return 0;
}

int vxn_model_validate(const vxn_model* m) { return static_cast<int>(voxanim::validate(*m->m).violations.size()); }

void vxn_model_free(vxn_model* m) { delete m; }

vxn_scene* vxn_scene_config(int config, vxn_model* const* models, uint32_t n_models, uint64_t seed, int width,
                            int height) {
    return guard(
        [&] {
            std::vector<std::shared_ptr<const voxanim::SvoModel>> ms;
            for (uint32_t i = 0; i < n_models; ++i) ms.push_back(models[i]->m);
            return new vxn_scene{voxanim::bench::make_config_scene(config, ms, seed, width, height)};
        },
        static_cast<vxn_scene*>(nullptr));
}

int vxn_scene_evaluate(vxn_scene* s, double time) {
    return guard(
        [&] {
            voxanim::evaluate_animation(s->s, time);
            return 0;
        },
        -1);
}

int vxn_scene_mark_clean(vxn_scene* s) {
    voxanim::mark_clean(s->s);
    return 0;
}

int vxn_scene_set_camera(vxn_scene* s, const double* pos, const double* at, const double* up, double fov, int width,
                         int height) {
    return guard(
        [&] {
            s->s.camera = voxanim::make_look_at_camera({pos[0], pos[1], pos[2]}, {at[0], at[1], at[2]},
                                                       {up[0], up[1], up[2]}, fov, width, height);
            s->s.camera.dirty = true;
            return 0;
        },
        -1);
}

int vxn_scene_set_camera_dirty(vxn_scene* s, int dirty) {
    s->s.camera.dirty = dirty != 0;
    return 0;
}

int vxn_scene_object_count(const vxn_scene* s) { return static_cast<int>(s->s.objects.size()); }

int vxn_scene_get_object(const vxn_scene* s, int index, int32_t* id, double* tf, int* dirty) {
    if (index < 0 || index >= static_cast<int>(s->s.objects.size())) return -1;
    const voxanim::SceneObject& o = s->s.objects[static_cast<std::size_t>(index)];
    if (id) *id = o.id;
    if (tf) std::memcpy(tf, &o.transform, sizeof(o.transform));
    if (dirty) *dirty = o.dirty ? 1 : 0;
    return 0;
}

int vxn_scene_set_object(vxn_scene* s, int index, const double* tf, int dirty) {
    if (index < 0 || index >= static_cast<int>(s->s.objects.size())) return -1;
    voxanim::SceneObject& o = s->s.objects[static_cast<std::size_t>(index)];
    if (tf) std::memcpy(static_cast<void*>(&o.transform), tf, sizeof(o.transform));
    o.dirty = dirty != 0;
    return 0;
}

namespace {

void export_frame(const voxanim::Scene& sc, vxa_frame_desc* f) {
    *f = vxa_frame_desc{};
    for (int k = 0; k < 3; ++k) f->camera.position[k] = sc.camera.position[k];
    std::memcpy(f->camera.orientation, sc.camera.orientation.m.data(), 9 * sizeof(double));
    f->camera.vertical_fov_deg = sc.camera.vertical_fov_deg;
    f->camera.width = sc.camera.width;
    f->camera.height = sc.camera.height;
    std::memcpy(f->background, sc.background.data(), 3);
    f->culling = 1;
    f->sorting = 1;
    f->camera_dirty = sc.camera.dirty ? 1 : 0;
    f->tile_rank = 0;
    f->tile_world = 1;
}

// Instances with model handles (one cache lookup per distinct model).
void export_instances(const voxanim::Scene& sc, vxa_instance* inst) {
    const voxanim::SvoModel* last = nullptr;
    std::uint32_t last_handle = 0;
    voxanim::gpu::begin_model_frame();
    for (std::size_t i = 0; i < sc.objects.size(); ++i) {
        const voxanim::SceneObject& o = sc.objects[i];
        vxa_instance& v = inst[i];
        v = vxa_instance{};
        v.id = o.id;
        if (o.model) {
            if (o.model.get() != last) {
                last = o.model.get();
                last_handle = voxanim::gpu::model_handle(o.model);
            }
            v.model = last_handle;
        }
        std::memcpy(v.rotation, o.transform.rotation.m.data(), 9 * sizeof(double));
        for (int k = 0; k < 3; ++k) {
            v.translation[k] = o.transform.translation[k];
            v.scale[k] = o.transform.scale[k];
        }
        v.dirty = o.dirty ? 1 : 0;
    }
}

} // namespace

int vxn_scene_submit(vxn_scene* s, double time, int precision, int rank, int world, uint32_t hbo_device) {
    return guard(
        [&] {
            if (time >= 0.0) voxanim::evaluate_animation(s->s, time);
            thread_local std::vector<vxa_instance> inst;
            inst.resize(s->s.objects.size());
            vxa_frame_desc f;
            export_frame(s->s, &f);
            export_instances(s->s, inst.data());
            f.precision = static_cast<std::uint8_t>(precision);
            f.tile_rank = rank;
            f.tile_world = world;
            f.hbo_device = hbo_device;
            voxanim::gpu::check(vxa_submit(voxanim::gpu::context(), &f, inst.data(),
                                           static_cast<std::uint32_t>(inst.size())),
                                "vxa_submit");
            voxanim::mark_clean(s->s); // the caller's per-frame mark_clean (reference cli.cpp:270)
            return 0;
        },
        -1);
}

int vxn_scene_stream(vxn_scene* s, double time, int precision, uint8_t* rgb_out, uint64_t* ticket) {
    return guard(
        [&] {
            if (time >= 0.0) voxanim::evaluate_animation(s->s, time);
            thread_local std::vector<vxa_instance> inst;
            inst.resize(s->s.objects.size());
            vxa_frame_desc f;
            export_frame(s->s, &f);
            export_instances(s->s, inst.data());
            f.precision = static_cast<std::uint8_t>(precision);
            voxanim::gpu::check(vxa_submit_readback(voxanim::gpu::context(), &f, inst.data(),
                                                    static_cast<std::uint32_t>(inst.size()), rgb_out, ticket),
                                "vxa_submit_readback");
            voxanim::mark_clean(s->s);
            return 0;
        },
        -1);
}

int vxn_scene_export(vxn_scene* s, vxa_frame_desc* f, vxa_instance* inst, uint32_t cap, uint32_t* count) {
    return guard(
        [&] {
            const voxanim::Scene& sc = s->s;
            if (count) *count = static_cast<uint32_t>(sc.objects.size());
            if (f) export_frame(sc, f);
            if (inst) {
                if (cap < sc.objects.size()) throw voxanim::ValidationError("export: instance buffer too small");
                export_instances(sc, inst);
            }
            return 0;
        },
        -1);
}

void vxn_scene_free(vxn_scene* s) { delete s; }

vxn_hbo* vxn_hbo_create(int width, int height) {
    return guard([&] { return new vxn_hbo{voxanim::HitBuffer(width, height)}; }, static_cast<vxn_hbo*>(nullptr));
}

void vxn_hbo_free(vxn_hbo* h) { delete h; }

int vxn_render(vxn_scene* s, int culling, int sorting, int precision, vxn_hbo* hbo, uint8_t* rgb, vxa_pixel_aov* aov,
               uint64_t* fs4, double* render_ms, vxa_stats* ds) {
    return guard(
        [&] {
            voxanim::RenderOptions opts;
            opts.culling = culling != 0;
            opts.sorting = sorting != 0;
            opts.hbo = hbo ? &hbo->b : nullptr;
            voxanim::gpu::RenderOptionsEx ex;
            ex.precision = precision < 0 ? voxanim::gpu::default_precision()
                                         : static_cast<voxanim::gpu::Precision>(precision);
            ex.read_image = rgb != nullptr;
            std::vector<vxa_pixel_aov> aovs;
            if (aov) ex.aov = &aovs;
            voxanim::FrameStats st;
            voxanim::gpu::render_frame_into(s->s, opts, ex, st, rgb, ds);
            if (aov) std::memcpy(aov, aovs.data(), aovs.size() * sizeof(vxa_pixel_aov));
            if (fs4) {
                fs4[0] = st.rays;
                fs4[1] = st.sphere_tests;
                fs4[2] = st.svo_traversals;
                fs4[3] = st.pixels_reused;
            }
            if (render_ms) *render_ms = st.render_ms;
            return 0;
        },
        -1);
}

int vxn_scene_render_image(vxn_scene* s, double time, int steps, double* ms_per_call, uint8_t* last_rgb) {
    return guard(
        [&] {
            voxanim::RenderOptions opts;
            voxanim::FrameStats st;
            double total = 0.0;
            for (int k = 0; k < steps; ++k) {
                voxanim::evaluate_animation(s->s, time + k / 30.0);
                const auto t0 = std::chrono::steady_clock::now();
                const voxanim::Image img = voxanim::render_frame(s->s, opts, st); // the drop-in call, by value
                total += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                voxanim::mark_clean(s->s);
                if (last_rgb && k == steps - 1) std::memcpy(last_rgb, img.rgb.data(), img.rgb.size());
            }
            if (ms_per_call) *ms_per_call = steps > 0 ? total / steps : 0.0;
            return 0;
        },
        -1);
}

int vxn_hbo_records(vxn_hbo* h, vxa_hit_record* out) {
    return guard(
        [&] {
            const voxanim::HitBuffer& b = h->b;
            std::memcpy(out, b.data(), sizeof(voxanim::HitRecord) * static_cast<std::size_t>(b.width()) * b.height());
            return 0;
        },
        -1);
}

int vxn_hbo_set_record(vxn_hbo* h, int x, int y, const vxa_hit_record* rec) {
    return guard(
        [&] {
            if (x < 0 || y < 0 || x >= h->b.width() || y >= h->b.height())
                throw voxanim::ValidationError("hit buffer index out of range");
            std::memcpy(static_cast<void*>(&h->b.at(x, y)), rec, sizeof(voxanim::HitRecord));
            return 0;
        },
        -1);
}

int vxn_traverse(const vxn_model* m, const vxa_local_ray* rays, uint32_t n, vxa_traverse_hit* hits) {
    return guard(
        [&] {
            const std::uint32_t h = voxanim::gpu::model_handle(*m->m);
            voxanim::gpu::check(vxa_traverse(voxanim::gpu::context(), h, rays, n, VXA_FP64, hits, nullptr, 0),
                                "vxa_traverse");
            return 0;
        },
        -1);
}

vxa_ctx* vxn_context(void) {
    return guard([&] { return voxanim::gpu::context(); }, static_cast<vxa_ctx*>(nullptr));
}

} // extern "C"
