// TEST INFRASTRUCTURE — the parity oracle. Not part of the product.
//
// Glue that exposes the REFERENCE implementation (proj/src/*.cpp compiled in
// place from /root/reference by oracle/Makefile into oracle/_ref/) through a
// flat C interface for tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg. Nothing in the product links this.
//
// What it provides, all computed by the reference's own functions:
//   * models: deserialize (svo.cpp:231-291), dense sphere / shell / random
//     grids -> build_from_grid (svo.cpp:80-132, ingest.cpp:193-266,
//     tests/support/oracles.hpp:265-279);
//   * scenes: bench_scenes.cpp compiled against the reference headers;
//     evaluate_animation (scene.cpp:370-385);
//   * frames: render_frame (renderer.cpp:218-300), timed by FrameStats::render_ms;
//   * per-pixel AOV dump: shade_pixel's candidate order and skip rule
//     (renderer.cpp:143-214, 63-100) replayed with traverse_debug so the hit
//     voxel (leaf_path_to_voxel), level (path_len), parent node and attribute
//     index (node_child replay, svo.cpp:27-39) and internal-node fetches are
//     known; its RGB must equal render_frame's image (checked by the tests);
//   * single rays: traverse / traverse_debug (traversal.cpp:249-258) and the
//     independent DDA oracle (oracles.hpp:68-149);
//   * the FP32 tie classifier (SURVEY.md §8(a) "Tie classification").
#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "support/oracles.hpp"
#include "voxanim/renderer.hpp"
#include "voxanim/scene.hpp"
#include "voxanim/svo.hpp"
#include "voxanim/traversal.hpp"

#include "bench_scenes.hpp"

using namespace voxanim;

struct vref_model {
    std::shared_ptr<const SvoModel> m;
};
struct vref_scene {
    Scene s;
};
struct vref_hbo {
    HitBuffer b;
};

// Same layouts as include/vxa.h (kept independent on purpose: the oracle does
// not include product headers).
struct AovRec {
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
static_assert(sizeof(AovRec) == 48);

struct LocalRayRec {
    double origin[3], direction[3], half_extent[3];
};
struct TravRec {
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
static_assert(sizeof(TravRec) == 96);

namespace {

thread_local std::string g_err;

template <class F> auto guard(F&& f, decltype(f()) on_error) -> decltype(f()) {
    try {
        return f();
    } catch (const std::exception& e) {
        g_err = e.what();
    } catch (...) {
        g_err = "unknown exception";
    }
    return on_error;
}

vref_model* wrap(SvoModel&& m) { return new vref_model{std::make_shared<const SvoModel>(std::move(m))}; }

int hw_threads(int t) {
    if (t > 0) return t;
    const int h = static_cast<int>(std::thread::hardware_concurrency());
    return h > 0 ? h : 1;
}

template <class F> void parallel_rows(int rows, int threads, F&& body) {
    threads = std::max(1, std::min(threads, rows));
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w) {
        const int a = static_cast<int>(static_cast<long long>(rows) * w / threads);
        const int b = static_cast<int>(static_cast<long long>(rows) * (w + 1) / threads);
        pool.emplace_back([&, a, b] { body(a, b); });
    }
    for (auto& t : pool) t.join();
}

// Replays node_child down a leaf path: parent node index and attribute index.
void replay_path(const SvoModel& m, const TraversalHit& h, uint32_t& parent, uint32_t& attr) {
    uint32_t node = 0;
    for (int l = 0; l + 1 < h.path_len; ++l) node = node_child(m, node, h.leaf_path[static_cast<std::size_t>(l)]).index;
    parent = node;
    attr = node_child(m, node, h.leaf_path[static_cast<std::size_t>(h.path_len - 1)]).index;
}

// Internal nodes fetched by one traversal = root (if the box is hit) + pushes.
uint32_t fetches_of(const SvoModel& m, const Ray& local, const OctreeBounds& b, const std::vector<TraversalVisit>& log) {
    if (!ray_box_params(local, b)) return 0;
    uint32_t n = 1;
    for (const TraversalVisit& v : log)
        if (!v.leaf && v.level < m.depth && v.level < kMaxTreeDepth) ++n;
    return n;
}

struct PixelOracle {
    AovRec aov{};
    std::array<std::uint8_t, 3> rgb{};
};

// shade_pixel without a hit buffer (renderer.cpp:143-214) + trace_ray (:63-100).
PixelOracle oracle_pixel(const Scene& scene, const std::vector<BoundingSphere>& spheres, const RenderOptions& opts,
                         const Ray& ray) {
    const bool sphere_pass = opts.culling || opts.sorting;
    std::vector<SphereHit> hits;
    if (sphere_pass) {
        for (std::size_t i = 0; i < scene.objects.size(); ++i)
            if (auto h = ray_sphere_test(ray, spheres[i])) {
                h->object_id = scene.objects[i].id;
                hits.push_back(*h);
            }
    }
    std::vector<SphereHit> cand;
    if (opts.culling) {
        cand = hits;
    } else {
        for (std::size_t i = 0; i < scene.objects.size(); ++i) {
            SphereHit e;
            e.object_id = scene.objects[i].id;
            if (opts.sorting) {
                if (auto h = ray_sphere_test(ray, spheres[i])) {
                    e.d = h->d;
                    e.t_center = h->t_center;
                    e.t_boundary = h->t_boundary;
                } else {
                    e.t_center = (spheres[i].center - ray.origin).dot(ray.direction);
                }
            }
            cand.push_back(e);
        }
    }
    if (opts.sorting) {
        std::sort(cand.begin(), cand.end(), [](const SphereHit& a, const SphereHit& b) {
            return a.t_center != b.t_center ? a.t_center < b.t_center : a.object_id < b.object_id;
        });
    } else {
        std::sort(cand.begin(), cand.end(), [](const SphereHit& a, const SphereHit& b) { return a.object_id < b.object_id; });
        for (auto& c : cand) c.t_boundary = 0.0;
    }

    PixelOracle out;
    HitRecord best;
    bool have = false;
    TraversalHit best_hit{};
    const SceneObject* best_obj = nullptr;
    uint32_t trav = 0, fetch = 0;
    for (const SphereHit& c : cand) {
        if (have && best.t < c.t_boundary) continue;
        const SceneObject* obj = scene.find_object(c.object_id);
        if (!obj || !obj->model) continue;
        const Ray local = transform_ray_world_to_local(ray, obj->transform);
        ++trav;
        const OctreeBounds b = bounds_from_scale(obj->transform.scale);
        std::vector<TraversalVisit> log;
        const auto hit = traverse_debug(*obj->model, local, b, log);
        fetch += fetches_of(*obj->model, local, b, log);
        if (!hit) continue;
        if (!have || hit->t_hit < best.t || (hit->t_hit == best.t && obj->id < best.object_id)) {
            have = true;
            best.color = hit->attribute;
            best.normal = obj->transform.rotation * hit->normal_local;
            best.t = hit->t_hit;
            best.object_id = obj->id;
            best_hit = *hit;
            best_obj = obj;
        }
    }
    if (have) best.kind = cand.size() > 1 ? HitKind::MultiSphere : HitKind::SingleSphere;
    out.rgb = shade(best, ray, scene.background);
    AovRec& a = out.aov;
    a.object_id = have ? best.object_id : -1;
    a.t = have ? best.t : 0.0;
    a.kind = static_cast<uint8_t>(best.kind);
    a.traversals = trav;
    a.node_fetches = fetch;
    if (have) {
        replay_path(*best_obj->model, best_hit, a.node_index, a.attr_index);
        const auto v = leaf_path_to_voxel(std::span<const std::uint8_t>(best_hit.leaf_path.data(), best_hit.path_len));
        a.voxel[0] = v[0];
        a.voxel[1] = v[1];
        a.voxel[2] = v[2];
        a.level = best_hit.path_len;
        a.entry_axis = best_hit.normal_local.x != 0.0 ? 0 : (best_hit.normal_local.y != 0.0 ? 1 : 2);
    }
    return out;
}

// ---- tie classification ----------------------------------------------------

constexpr double kInf = std::numeric_limits<double>::infinity();

double tau(double t) { return 8.0 * std::ldexp(1.0, -23) * std::max(1.0, std::abs(t)); }

// FP32 error of a plane parameter on local axis a of the instance: the plane's
// position is resolved to 2^-22 of (|o_a| + 2 h_a) (origin and cell size
// rounded to FP32), which moves t by that over the incidence |d_a| -- large on a
// grazing axis. Capped at the larger of 2^-12 of t and `extent` (the t-extent
// of the voxel in question along the ray, when the caller has one): a nearly
// parallel plane can put t anywhere in that voxel's stretch of the ray (a 5600-
// scene soak found one such pixel, |d_a| = 3.6e-5, 1.5 % off in t, right voxel),
// but not beyond it.
double plane_err(const SceneObject& obj, const Ray& world, int a, double t, double extent = 0.0) {
    if (a < 0) return 0.0;
    const Ray loc = transform_ray_world_to_local(world, obj.transform);
    const double da = std::abs(loc.direction[a]);
    const double cap = std::max(std::ldexp(std::max(1.0, std::abs(t)), -12), extent);
    if (da == 0.0) return 0.0;
    const double h = bounds_from_scale(obj.transform.scale).half_extent[a];
    return std::min(std::ldexp(std::abs(loc.origin[a]) + 2.0 * h, -22) / da, cap);
}

struct Interval {
    double in = kInf, out = -kInf;
    double axis_in[3] = {-kInf, -kInf, -kInf}; // entry parameter of each axis' slab
    int in_axis = -1, out_axis = -1;           // the axes whose planes give in / out
};

// FP64 slab test of the voxel box (level `level` of the instance's octree)
// against the local ray.
Interval voxel_interval(const SceneObject& obj, const Ray& world, const uint32_t v[3], uint32_t level) {
    const Ray r = transform_ray_world_to_local(world, obj.transform);
    const OctreeBounds b = bounds_from_scale(obj.transform.scale);
    Interval iv{-kInf, kInf};
    for (int a = 0; a < 3; ++a) {
        const double h = b.half_extent[a];
        const double cell = 2.0 * h / std::ldexp(1.0, static_cast<int>(level));
        const double lo = -h + v[a] * cell, hi = lo + cell;
        const double o = r.origin[a], d = r.direction[a];
        if (d == 0.0) {
            if (o < lo || o >= hi) return {kInf, -kInf};
            continue;
        }
        double t0 = (lo - o) / d, t1 = (hi - o) / d;
        if (t0 > t1) std::swap(t0, t1);
        iv.axis_in[a] = t0;
        if (t0 > iv.in) iv.in = t0, iv.in_axis = a;
        if (t1 < iv.out) iv.out = t1, iv.out_axis = a;
    }
    return iv;
}

// A zero-direction axis whose origin lies on (or within FP32 resolution of)
// one of the voxel's boundary planes: the ray runs along the face between two
// voxel rows, and which row owns it is the half-open convention's tie.
bool on_zero_dir_face(const SceneObject& obj, const Ray& world, const uint32_t v[3], uint32_t level) {
    const Ray r = transform_ray_world_to_local(world, obj.transform);
    const OctreeBounds b = bounds_from_scale(obj.transform.scale);
    for (int a = 0; a < 3; ++a) {
        if (std::abs(r.direction[a]) > 1e-6) continue;
        const double h = b.half_extent[a];
        const double cell = 2.0 * h / std::ldexp(1.0, static_cast<int>(level));
        const double lo = -h + v[a] * cell, hi = lo + cell;
        const double eps = std::ldexp(std::abs(r.origin[a]) + 2.0 * h, -20);
        if (std::abs(r.origin[a] - lo) <= eps || std::abs(r.origin[a] - hi) <= eps) return true;
    }
    return false;
}

bool sphere_grazed(const SceneObject& obj, const Ray& ray, double t_ref) {
    const BoundingSphere s = bounding_sphere(obj);
    const Vec3 l = s.center - ray.origin;
    const double tc = l.dot(ray.direction);
    const double d2 = l.norm2() - tc * tc;
    const double r2 = s.radius * s.radius;
    return std::abs(d2 - r2) <= tau(t_ref) * std::max(1.0, r2) * 16.0;
}

bool box_grazed(const SceneObject& obj, const Ray& world, double t_ref) {
    const Ray r = transform_ray_world_to_local(world, obj.transform);
    const OctreeBounds b = bounds_from_scale(obj.transform.scale);
    double tin = -kInf, tout = kInf;
    for (int a = 0; a < 3; ++a) {
        const double h = b.half_extent[a], o = r.origin[a], d = r.direction[a];
        if (d == 0.0) {
            if (std::abs(o - h) <= tau(t_ref) || std::abs(o + h) <= tau(t_ref)) return true;
            continue;
        }
        double t0 = (-h - o) / d, t1 = (h - o) / d;
        if (t0 > t1) std::swap(t0, t1);
        tin = std::max(tin, t0);
        tout = std::min(tout, t1);
    }
    return std::abs(tout - tin) <= tau(t_ref) || std::abs(tout) <= tau(t_ref);
}

// FP64 entry parameter of an instance for this ray (reference traverse).
bool instance_t(const SceneObject& obj, const Ray& world, double& t) {
    if (!obj.model) return false;
    const Ray local = transform_ray_world_to_local(world, obj.transform);
    const auto h = traverse(*obj.model, local, bounds_from_scale(obj.transform.scale));
    if (!h) return false;
    t = h->t_hit;
    return true;
}

// Per-pixel classification of an FP32 result against the oracle's, by rule
// (the tie rules are geometric: each names the FP64 near-coincidence that lets
// an FP32 traversal legitimately pick the other answer). Every rule's share is
// reported per frame (vref_classify_rules) so no rule can silently absorb bugs.
enum Rule : int {
    kMatch = 0,
    kTieEntryFace = 1,    // same voxel, entered through another face at an edge/corner (entry planes within tau)
    kTieSphereGraze = 2,  // a bounding sphere grazed (|d^2 - r^2| small): candidate sets may differ
    kTieBoxGraze = 3,     // an instance's root box grazed
    kTieZeroDirFace = 4,  // a zero-direction axis running along a voxel face (half-open convention)
    kTieOracleGrazed = 5, // the oracle's voxel is only grazed (t_out - t_in <= tau)
    kTieGpuNearMiss = 6,  // the GPU's voxel is a near miss / graze (|t_in - t_out| <= tau)
    kTieBehindOrigin = 7, // the GPU's voxel ends within tau behind the origin
    kTieSameEntry = 8,    // both voxels (different ones) entered at the same parameter (within tau)
    kTieInstance = 9,     // two instances' FP64 hits within tau (nearest (t, id) selection)
    kTieMissGraze = 10,   // GPU missed; the oracle's voxel is nearly grazed (within 4 tau)
    kRuleCount = 11,
    kBug = 100,           // unexplained difference
    kTOutOfTol = 101,     // same hit, t outside the stated FP32 tolerance
};

// The t tolerance of a matching hit: t_rel relative, plus the FP32 error of the
// entry planes the two answers used (plane_err: a grazing entry is
// ill-conditioned), each capped at the larger of 2^-12 of t and the voxel's
// t-extent along the ray.
double t_tolerance(const Scene& scene, const Ray& ray, const AovRec& o, const AovRec& g, double t_rel) {
    const SceneObject* obj = scene.find_object(o.object_id);
    const Interval iv = voxel_interval(*obj, ray, o.voxel, o.level);
    const double ext = iv.out > iv.in ? iv.out - iv.in : 0.0;
    return t_rel * std::max(1.0, std::abs(o.t)) +
           std::max(plane_err(*obj, ray, o.entry_axis, o.t, ext), plane_err(*obj, ray, g.entry_axis, o.t, ext));
}

// Replays node_child (svo.cpp:27-39) along the voxel's octant path: true iff a
// leaf sits exactly there, with its parent node and attribute index.
bool leaf_at(const SvoModel& m, const uint32_t v[3], uint32_t level, uint32_t& parent, uint32_t& attr) {
    if (level < 1 || level > m.depth || m.nodes.empty()) return false;
    uint32_t node = 0;
    for (uint32_t l = 0; l < level; ++l) {
        const uint32_t sh = level - 1 - l;
        const unsigned oct = (((v[0] >> sh) & 1u) << 2) | (((v[1] >> sh) & 1u) << 1) | ((v[2] >> sh) & 1u);
        const ChildRef c = node_child(m, node, oct);
        if (c.absent()) return false;
        if (c.is_leaf()) {
            if (l + 1 != level) return false;
            parent = node;
            attr = c.index;
            return true;
        }
        node = c.index;
    }
    return false;
}

// Every near-coincidence test below allows tau (8 FP32 ulp of t) plus the FP32
// plane errors (plane_err) of the axes whose planes the compared parameters come
// from -- an FP32 traversal can only disagree with FP64 by that much.
int classify_rule(const Scene& scene, const Ray& ray, const AovRec& o, const AovRec& g, double t_rel) {
    const bool ho = o.object_id >= 0, hg = g.object_id >= 0;
    if (!ho && !hg) return kMatch;
    const bool same_voxel = ho && hg && o.object_id == g.object_id && o.voxel[0] == g.voxel[0] &&
                            o.voxel[1] == g.voxel[1] && o.voxel[2] == g.voxel[2] && o.level == g.level;
    if (same_voxel) {
        // the leaf's parent node and attribute are functions of its path: the same
        // voxel with another node or attribute index is a bug, never a tie
        if (o.node_index != g.node_index || o.attr_index != g.attr_index) return kBug;
        if (std::abs(o.t - g.t) > t_tolerance(scene, ray, o, g, t_rel)) return kTOutOfTol;
        if (o.entry_axis == g.entry_axis) return kMatch;
        const SceneObject* obj = scene.find_object(o.object_id);
        const Interval iv = voxel_interval(*obj, ray, o.voxel, o.level);
        const double tol = tau(o.t) + plane_err(*obj, ray, o.entry_axis, o.t) + plane_err(*obj, ray, g.entry_axis, o.t);
        return std::abs(iv.axis_in[o.entry_axis] - iv.axis_in[g.entry_axis]) <= tol ? kTieEntryFace : kBug;
    }
    const double tref = ho ? o.t : g.t;
    const double tt = tau(tref);
    const SceneObject* oo = ho ? scene.find_object(o.object_id) : nullptr;
    const SceneObject* og = hg ? scene.find_object(g.object_id) : nullptr;
    const auto err2 = [&](const SceneObject* obj, const Interval& v) {
        return plane_err(*obj, ray, v.in_axis, tref) + plane_err(*obj, ray, v.out_axis, tref);
    };
    if (hg) {
        // Whatever the GPU hit must be a real answer for this ray: an existing
        // leaf of its instance's model (with that leaf's parent node and
        // attribute), on the ray, entered at the GPU's t. The tie rules below
        // only decide whether choosing it over the oracle's leaf is explained by
        // an FP64 near-coincidence.
        if (og == nullptr || !og->model) return kBug;
        uint32_t parent = 0, attr = 0;
        if (!leaf_at(*og->model, g.voxel, g.level, parent, attr)) return kBug;
        if (parent != g.node_index || attr != g.attr_index) return kBug;
        // (a ray running along a face on a zero-direction axis belongs to either
        // side: the half-open convention's tie, checked below)
        if (!on_zero_dir_face(*og, ray, g.voxel, g.level)) {
            const Interval v = voxel_interval(*og, ray, g.voxel, g.level);
            const double tol = tt + err2(og, v);
            if (v.in - v.out > tol) return kBug; // the ray does not pass through it
            if (v.out < -tol) return kBug;       // wholly behind the origin
            const double t_in = std::max(v.in, 0.0);
            const double ext = v.out > v.in ? v.out - v.in : 0.0;
            if (std::abs(g.t - t_in) > tt + t_rel * std::max(1.0, t_in) + plane_err(*og, ray, v.in_axis, t_in, ext) +
                                           plane_err(*og, ray, g.entry_axis, t_in, ext))
                return kBug; // not entered at the GPU's t
        }
    }
    if (ho && hg && o.object_id == g.object_id && o.level != g.level) {
        // a leaf never contains another leaf: the GPU's voxel being an ancestor or a
        // descendant of the oracle's (a traversal stopping early or late) is a bug
        const uint32_t lo = std::min(o.level, g.level), hi = std::max(o.level, g.level);
        const uint32_t* vlo = o.level < g.level ? o.voxel : g.voxel;
        const uint32_t* vhi = o.level < g.level ? g.voxel : o.voxel;
        if ((vhi[0] >> (hi - lo)) == vlo[0] && (vhi[1] >> (hi - lo)) == vlo[1] && (vhi[2] >> (hi - lo)) == vlo[2])
            return kBug;
    }
    for (const SceneObject* obj : {oo, og})
        if (obj && sphere_grazed(*obj, ray, tref)) return kTieSphereGraze;
    for (const SceneObject* obj : {oo, og})
        if (obj && box_grazed(*obj, ray, tref)) return kTieBoxGraze;
    if ((oo && on_zero_dir_face(*oo, ray, o.voxel, o.level)) || (og && on_zero_dir_face(*og, ray, g.voxel, g.level)))
        return kTieZeroDirFace;
    Interval vo, vg;
    if (oo) {
        vo = voxel_interval(*oo, ray, o.voxel, o.level);
        if (vo.out - vo.in <= tt + err2(oo, vo)) return kTieOracleGrazed;
    }
    if (og) {
        vg = voxel_interval(*og, ray, g.voxel, g.level);
        const double tol = tt + err2(og, vg);
        if (std::abs(vg.in - vg.out) <= tol) return kTieGpuNearMiss;
        if (vg.out < 0.0 && vg.out > -tol) return kTieBehindOrigin;
        // a GPU voxel the ray does not pass through at all is a bug whatever else holds
        if (vg.in > vg.out) return kBug;
    }
    if (oo && og) {
        const double ti = std::max(vo.in, 0.0), tg = std::max(vg.in, 0.0);
        const double tol = tt + plane_err(*oo, ray, vo.in_axis, tref) + plane_err(*og, ray, vg.in_axis, tref);
        if (std::abs(ti - tg) <= tol) return kTieSameEntry;
        if (o.object_id != g.object_id) {
            double t64 = 0.0;
            if (instance_t(*og, ray, t64) && std::abs(t64 - o.t) <= tol) return kTieInstance;
        }
    }
    if (!hg && oo && vo.out - vo.in <= 4 * tt + err2(oo, vo)) return kTieMissGraze;
    return kBug;
}

// 0: equal; 1: documented slab-test tie; 2: unexplained (a bug); 3: same hit but t out of tolerance.
int classify_pixel(const Scene& scene, const Ray& ray, const AovRec& o, const AovRec& g, double t_rel) {
    const int r = classify_rule(scene, ray, o, g, t_rel);
    return r == kMatch ? 0 : r == kBug ? 2 : r == kTOutOfTol ? 3 : 1;
}

} // namespace

#define VREF_API __attribute__((visibility("default")))

extern "C" {

VREF_API const char* vref_last_error(void) { return g_err.c_str(); }

VREF_API vref_model* vref_model_deserialize(const uint8_t* bytes, size_t n) {
    return guard([&] { return wrap(deserialize(std::span<const std::uint8_t>(bytes, n))); }, (vref_model*)nullptr);
}

// The reference's own file loader (svo.cpp: load_svo -> deserialize).
VREF_API vref_model* vref_model_load(const char* path) {
    return guard([&] { return wrap(load_svo(path)); }, (vref_model*)nullptr);
}

VREF_API vref_model* vref_model_dense_sphere(uint32_t depth) {
    return guard([&] { return wrap(build_from_grid(gen_primitive(PrimitiveKind::Sphere, depth), depth)); },
                 (vref_model*)nullptr);
}

// Shell of the reference's sphere: solid voxels with a 6-neighbour outside the
// solid or outside the grid.
VREF_API vref_model* vref_model_shell_grid(uint32_t depth) {
    return guard(
        [&] {
            const VoxelGrid solid = gen_primitive(PrimitiveKind::Sphere, depth);
            const int n = static_cast<int>(solid.resolution());
            VoxelGrid shell(solid.resolution());
            const auto in = [&](int x, int y, int z) {
                return x >= 0 && y >= 0 && z >= 0 && x < n && y < n && z < n &&
                       solid.is_set(static_cast<uint32_t>(x), static_cast<uint32_t>(y), static_cast<uint32_t>(z));
            };
            for (int x = 0; x < n; ++x)
                for (int y = 0; y < n; ++y)
                    for (int z = 0; z < n; ++z)
                        if (in(x, y, z) && !(in(x - 1, y, z) && in(x + 1, y, z) && in(x, y - 1, z) && in(x, y + 1, z) &&
                                             in(x, y, z - 1) && in(x, y, z + 1)))
                            shell.set(static_cast<uint32_t>(x), static_cast<uint32_t>(y), static_cast<uint32_t>(z));
            return wrap(build_from_grid(shell, depth));
        },
        (vref_model*)nullptr);
}

// The reference's own build_from_grid (svo.cpp:80-132) on a caller-supplied
// VoxelGrid bitset (x-major, (n^3+63)/64 words) and ColorSpec.
VREF_API vref_model* vref_model_from_grid(const uint64_t* words, uint32_t depth, uint32_t color_mode, uint32_t rgba) {
    return guard(
        [&] {
            ColorSpec cs;
            cs.mode = static_cast<ColorMode>(color_mode);
            cs.constant = {static_cast<uint8_t>(rgba), static_cast<uint8_t>(rgba >> 8), static_cast<uint8_t>(rgba >> 16),
                           static_cast<uint8_t>(rgba >> 24)};
            const uint32_t n = 1u << depth;
            VoxelGrid g(n, cs);
            const uint64_t bits = uint64_t{n} * n * n;
            for (uint64_t w = 0; w < (bits + 63) / 64; ++w)
                for (uint64_t v = words[w]; v; v &= v - 1) {
                    const uint64_t i = 64 * w + static_cast<uint64_t>(__builtin_ctzll(v));
                    if (i >= bits) break;
                    g.set(static_cast<uint32_t>(i / (uint64_t{n} * n)), static_cast<uint32_t>((i / n) % n),
                          static_cast<uint32_t>(i % n));
                }
            return wrap(build_from_grid(g, depth));
        },
        (vref_model*)nullptr);
}

VREF_API vref_model* vref_model_random(uint64_t seed, uint32_t depth, double fill) {
    return guard(
        [&] {
            std::mt19937_64 rng(seed);
            return wrap(build_from_grid(oracles::random_grid(rng, depth, fill), depth));
        },
        (vref_model*)nullptr);
}

VREF_API int vref_model_validate(const vref_model* m) {
    return static_cast<int>(validate(*m->m).violations.size());
}

VREF_API int64_t vref_model_serialize(const vref_model* m, uint8_t* out, size_t cap) {
    return guard(
        [&]() -> int64_t {
            const auto b = serialize(*m->m);
            if (out) {
                if (cap < b.size()) throw ValidationError("buffer too small");
                std::memcpy(out, b.data(), b.size());
            }
            return static_cast<int64_t>(b.size());
        },
        int64_t{-1});
}

VREF_API void vref_model_free(vref_model* m) { delete m; }

VREF_API vref_scene* vref_scene_config(int config, vref_model* const* models, uint32_t n, uint64_t seed, int w, int h) {
    return guard(
        [&] {
            std::vector<std::shared_ptr<const SvoModel>> ms;
            for (uint32_t i = 0; i < n; ++i) ms.push_back(models[i]->m);
            return new vref_scene{bench::make_config_scene(config, ms, seed, w, h)};
        },
        (vref_scene*)nullptr);
}

VREF_API int vref_scene_evaluate(vref_scene* s, double t) {
    return guard(
        [&] {
            evaluate_animation(s->s, t);
            return 0;
        },
        -1);
}

VREF_API int vref_scene_mark_clean(vref_scene* s) {
    mark_clean(s->s);
    return 0;
}

VREF_API int vref_scene_set_camera(vref_scene* s, const double* pos, const double* at, const double* up, double fov,
                                   int width, int height) {
    return guard(
        [&] {
            s->s.camera = make_look_at_camera({pos[0], pos[1], pos[2]}, {at[0], at[1], at[2]}, {up[0], up[1], up[2]},
                                              fov, width, height);
            s->s.camera.dirty = true;
            return 0;
        },
        -1);
}

VREF_API int vref_scene_set_camera_dirty(vref_scene* s, int dirty) {
    s->s.camera.dirty = dirty != 0;
    return 0;
}

VREF_API int vref_scene_get_object(const vref_scene* s, int index, int32_t* id, double* tf, int* dirty) {
    if (index < 0 || index >= static_cast<int>(s->s.objects.size())) return -1;
    const SceneObject& o = s->s.objects[static_cast<std::size_t>(index)];
    if (id) *id = o.id;
    if (tf) std::memcpy(tf, static_cast<const void*>(&o.transform), sizeof(o.transform));
    if (dirty) *dirty = o.dirty ? 1 : 0;
    return 0;
}

VREF_API int vref_scene_set_object(vref_scene* s, int index, const double* tf, int dirty) {
    if (index < 0 || index >= static_cast<int>(s->s.objects.size())) return -1;
    SceneObject& o = s->s.objects[static_cast<std::size_t>(index)];
    if (tf) std::memcpy(static_cast<void*>(&o.transform), tf, sizeof(o.transform));
    o.dirty = dirty != 0;
    return 0;
}

VREF_API void vref_scene_free(vref_scene* s) { delete s; }

VREF_API vref_hbo* vref_hbo_create(int w, int h) {
    return guard([&] { return new vref_hbo{HitBuffer(w, h)}; }, (vref_hbo*)nullptr);
}

VREF_API void vref_hbo_free(vref_hbo* h) { delete h; }

// The reference HitBuffer's records, read and written through at() (48-byte HitRecord layout).
VREF_API int vref_hbo_records(const vref_hbo* h, uint8_t* out) {
    const int w = h->b.width(), hh = h->b.height();
    for (int y = 0; y < hh; ++y)
        for (int x = 0; x < w; ++x)
            std::memcpy(out + 48 * (static_cast<size_t>(y) * w + x), &h->b.at(x, y), 48);
    return 0;
}
VREF_API int vref_hbo_set_record(vref_hbo* h, int x, int y, const uint8_t* rec) {
    std::memcpy(&h->b.at(x, y), rec, 48);
    return 0;
}

// The reference frame: render_frame with its own timing (FrameStats::render_ms).
VREF_API int vref_render(vref_scene* s, int culling, int sorting, int threads, vref_hbo* hbo, uint8_t* rgb, uint64_t* fs4,
                double* render_ms) {
    return guard(
        [&] {
            RenderOptions opts;
            opts.culling = culling != 0;
            opts.sorting = sorting != 0;
            opts.threads = threads;
            opts.hbo = hbo ? &hbo->b : nullptr;
            FrameStats st;
            const Image img = render_frame(s->s, opts, st);
            if (rgb) std::memcpy(rgb, img.rgb.data(), img.rgb.size());
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

// The reference's per-pixel work of render_frame (no hit buffer) restricted to
// rows [row_begin, row_end): generate_primary_ray, the sphere pass over
// per-frame bounding spheres, (t_center, id) order, the reference trace_ray
// and shade -- a bounded sample of a frame for the CPU baseline. Returns the
// wall time in ms through *ms.
VREF_API int vref_render_rows(const vref_scene* s, int threads, int row_begin, int row_end, uint8_t* rgb, double* ms) {
    return guard(
        [&] {
            const auto t0 = std::chrono::steady_clock::now();
            const Scene& scene = s->s;
            const int W = scene.camera.width;
            std::vector<BoundingSphere> spheres;
            for (const SceneObject& o : scene.objects) spheres.push_back(bounding_sphere(o));
            parallel_rows(row_end - row_begin, hw_threads(threads), [&](int a, int b) {
                std::vector<SphereHit> cand;
                for (int r = a; r < b; ++r) {
                    const int py = row_begin + r;
                    for (int px = 0; px < W; ++px) {
                        const Ray ray = generate_primary_ray(scene.camera, px, py);
                        cand.clear();
                        for (std::size_t i = 0; i < scene.objects.size(); ++i)
                            if (auto h = ray_sphere_test(ray, spheres[i])) {
                                h->object_id = scene.objects[i].id;
                                cand.push_back(*h);
                            }
                        std::sort(cand.begin(), cand.end(), [](const SphereHit& x, const SphereHit& y) {
                            return x.t_center != y.t_center ? x.t_center < y.t_center : x.object_id < y.object_id;
                        });
                        const HitRecord rec = trace_ray(scene, ray, cand, nullptr);
                        const auto c = shade(rec, ray, scene.background);
                        if (rgb) std::memcpy(rgb + 3 * (static_cast<std::size_t>(r) * W + px), c.data(), 3);
                    }
                }
            });
            *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            return 0;
        },
        -1);
}

// Per-pixel oracle over the rows [row_begin, row_end) (whole frame if both 0).
VREF_API int vref_dump(const vref_scene* s, int culling, int sorting, int threads, int row_begin, int row_end, AovRec* aov,
              uint8_t* rgb) {
    return guard(
        [&] {
            const Scene& scene = s->s;
            const int W = scene.camera.width;
            if (row_begin == 0 && row_end == 0) row_end = scene.camera.height;
            RenderOptions opts;
            opts.culling = culling != 0;
            opts.sorting = sorting != 0;
            std::vector<BoundingSphere> spheres;
            for (const SceneObject& o : scene.objects) spheres.push_back(bounding_sphere(o));
            parallel_rows(row_end - row_begin, hw_threads(threads), [&](int a, int b) {
                for (int r = a; r < b; ++r) {
                    const int py = row_begin + r;
                    for (int px = 0; px < W; ++px) {
                        const PixelOracle po = oracle_pixel(scene, spheres, opts, generate_primary_ray(scene.camera, px, py));
                        const std::size_t i = static_cast<std::size_t>(r) * W + px;
                        if (aov) aov[i] = po.aov;
                        if (rgb) std::memcpy(rgb + 3 * i, po.rgb.data(), 3);
                    }
                }
            });
            return 0;
        },
        -1);
}

// Tie classification of GPU AOVs against oracle AOVs (rows as in vref_dump).
VREF_API int vref_classify(const vref_scene* s, int row_begin, int row_end, const AovRec* oracle, const AovRec* gpu,
                  double t_rel, uint8_t* cls) {
    return guard(
        [&] {
            const Scene& scene = s->s;
            const int W = scene.camera.width;
            for (int py = row_begin; py < row_end; ++py)
                for (int px = 0; px < W; ++px) {
                    const std::size_t i = static_cast<std::size_t>(py - row_begin) * W + px;
                    cls[i] = static_cast<uint8_t>(
                        classify_pixel(scene, generate_primary_ray(scene.camera, px, py), oracle[i], gpu[i], t_rel));
                }
            return 0;
        },
        -1);
}

// Human-readable breakdown of one pixel's classification (debugging aid).
// Rule codes (classify_rule) per pixel of rows [row_begin, row_end).
VREF_API int vref_classify_rules(const vref_scene* s, int row_begin, int row_end, const AovRec* oracle,
                                 const AovRec* gpu, double t_rel, uint8_t* out) {
    return guard(
        [&] {
            const Scene& scene = s->s;
            const int W = scene.camera.width;
            for (int py = row_begin; py < row_end; ++py)
                for (int px = 0; px < W; ++px) {
                    const size_t i = static_cast<size_t>(py - row_begin) * W + px;
                    out[i] = static_cast<uint8_t>(
                        classify_rule(scene, generate_primary_ray(scene.camera, px, py), oracle[i], gpu[i], t_rel));
                }
            return 0;
        },
        -1);
}

VREF_API int vref_explain(const vref_scene* s, int px, int py, const AovRec* o, const AovRec* g, char* buf, size_t n) {
    return guard(
        [&] {
            const Scene& scene = s->s;
            const Ray ray = generate_primary_ray(scene.camera, px, py);
            std::string out;
            char line[512];
            const auto add = [&](const char* fmt, auto... a) {
                std::snprintf(line, sizeof(line), fmt, a...);
                out += line;
            };
            add("pixel (%d,%d) dir (%.17g %.17g %.17g)\n", px, py, ray.direction.x, ray.direction.y, ray.direction.z);
            for (const AovRec* r : {o, g}) {
                add("  %s: id %d t %.17g voxel (%u %u %u) level %u axis %u node %u attr %u trav %u fetch %u\n",
                    r == o ? "oracle" : "gpu   ", r->object_id, r->t, r->voxel[0], r->voxel[1], r->voxel[2],
                    r->level, r->entry_axis, r->node_index, r->attr_index, r->traversals, r->node_fetches);
                if (r->object_id >= 0) {
                    const SceneObject* obj = scene.find_object(r->object_id);
                    const Interval iv = voxel_interval(*obj, ray, r->voxel, r->level);
                    const Ray loc = transform_ray_world_to_local(ray, obj->transform);
                    add("    voxel interval [%.17g, %.17g] len %.3g  local d (%.6g %.6g %.6g) o (%.6g %.6g %.6g)\n",
                        iv.in, iv.out, iv.out - iv.in, loc.direction.x, loc.direction.y, loc.direction.z, loc.origin.x,
                        loc.origin.y, loc.origin.z);
                    double t64 = 0;
                    if (instance_t(*obj, ray, t64)) add("    fp64 traverse t %.17g\n", t64);
                    uint32_t par = 0, at = 0;
                    const bool leaf = obj->model && leaf_at(*obj->model, r->voxel, r->level, par, at);
                    add("    leaf_at %d parent %u attr %u  t - max(in,0) = %.3g  sphere_grazed %d box_grazed %d zero_face %d\n",
                        leaf ? 1 : 0, par, at, r->t - std::max(iv.in, 0.0), sphere_grazed(*obj, ray, r->t) ? 1 : 0,
                        box_grazed(*obj, ray, r->t) ? 1 : 0, on_zero_dir_face(*obj, ray, r->voxel, r->level) ? 1 : 0);
                }
            }
            add("  tau %.3g class %d rule %d\n", tau(o->object_id >= 0 ? o->t : g->t),
                classify_pixel(scene, ray, *o, *g, 1e-6), classify_rule(scene, ray, *o, *g, 1e-6));
            std::snprintf(buf, n, "%s", out.c_str());
            return 0;
        },
        -1);
}

// Reference traverse (+ optional visit log) for a batch of local rays.
VREF_API int vref_traverse(const vref_model* m, const LocalRayRec* rays, uint32_t n, TravRec* out, int with_fetches) {
    return guard(
        [&] {
            for (uint32_t i = 0; i < n; ++i) {
                const Ray r{{rays[i].origin[0], rays[i].origin[1], rays[i].origin[2]},
                            {rays[i].direction[0], rays[i].direction[1], rays[i].direction[2]}};
                const OctreeBounds b{{rays[i].half_extent[0], rays[i].half_extent[1], rays[i].half_extent[2]}};
                std::vector<TraversalVisit> log;
                const auto h = with_fetches ? traverse_debug(*m->m, r, b, log) : traverse(*m->m, r, b);
                TravRec t{};
                t.log_total = static_cast<uint32_t>(log.size());
                if (with_fetches) t.node_fetches = fetches_of(*m->m, r, b, log);
                if (h) {
                    t.hit = 1;
                    t.t_hit = h->t_hit;
                    t.t_enter = h->t_enter;
                    t.t_exit = h->t_exit;
                    t.normal_local[0] = h->normal_local.x;
                    t.normal_local[1] = h->normal_local.y;
                    t.normal_local[2] = h->normal_local.z;
                    t.attribute[0] = h->attribute.r;
                    t.attribute[1] = h->attribute.g;
                    t.attribute[2] = h->attribute.b;
                    t.attribute[3] = h->attribute.a;
                    std::copy(h->leaf_path.begin(), h->leaf_path.end(), t.leaf_path);
                    t.path_len = h->path_len;
                    replay_path(*m->m, *h, t.node_index, t.attr_index);
                }
                out[i] = t;
            }
            return 0;
        },
        -1);
}

// Independent DDA oracle on the random grid (seed, depth, fill): voxel + t per ray.
VREF_API int vref_dda_random(uint64_t seed, uint32_t depth, double fill, const LocalRayRec* rays, uint32_t n, int32_t* hit,
                    uint32_t* voxel, double* t) {
    return guard(
        [&] {
            std::mt19937_64 rng(seed);
            const VoxelGrid g = oracles::random_grid(rng, depth, fill);
            for (uint32_t i = 0; i < n; ++i) {
                const Ray r{{rays[i].origin[0], rays[i].origin[1], rays[i].origin[2]},
                            {rays[i].direction[0], rays[i].direction[1], rays[i].direction[2]}};
                const Vec3 h{rays[i].half_extent[0], rays[i].half_extent[1], rays[i].half_extent[2]};
                const auto d = oracles::dda_trace(g, h, r);
                hit[i] = d ? 1 : 0;
                if (d) {
                    voxel[3 * i] = d->x;
                    voxel[3 * i + 1] = d->y;
                    voxel[3 * i + 2] = d->z;
                    t[i] = d->t;
                }
            }
            return 0;
        },
        -1);
}

// The reference's primary ray for a pixel (renderer.cpp:11-23): origin, direction.
VREF_API int vref_primary_ray(const vref_scene* s, int px, int py, double* o6) {
    return guard(
        [&] {
            const Ray r = generate_primary_ray(s->s.camera, px, py);
            o6[0] = r.origin.x, o6[1] = r.origin.y, o6[2] = r.origin.z;
            o6[3] = r.direction.x, o6[4] = r.direction.y, o6[5] = r.direction.z;
            return 0;
        },
        -1);
}

VREF_API int vref_hardware_threads(void) { return hw_threads(0); }

} // extern "C"
