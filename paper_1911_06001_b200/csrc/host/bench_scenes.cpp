// Scene definitions for the benchmark configurations; see bench_scenes.hpp.
// Compiled twice: into libvoxanim (this repo's API) and into the reference
// harness (oracle/_ref, against /root/reference/proj/include).
#include "bench_scenes.hpp"

#include <cmath>
#include <numbers>
#include <random>
#include <stdexcept>

namespace voxanim::bench {

namespace {

constexpr double kPi = std::numbers::pi;

Quaternion axis_angle_deg(const Vec3& axis, double deg) { return Quaternion::from_axis_angle(axis, deg * kPi / 180.0); }

RigidTransform transform_of(const Keyframe& k) {
    RigidTransform tf;
    tf.rotation = rotation_from_quaternion(k.rotation);
    tf.translation = k.translation;
    tf.scale = k.scale;
    return tf;
}

SceneObject object(std::int32_t id, const std::shared_ptr<const SvoModel>& model, const RigidTransform& tf) {
    SceneObject o;
    o.id = id;
    o.model_name = "m" + std::to_string(id);
    o.model = model;
    o.transform = tf;
    o.dirty = false;
    return o;
}

// Normalised standard-normal 3-vector (method of the reference test oracles).
Vec3 unit_normal3(std::mt19937_64& rng) {
    std::normal_distribution<double> g(0.0, 1.0);
    while (true) {
        const Vec3 v{g(rng), g(rng), g(rng)};
        const double n = v.norm();
        if (n > 1e-6) return {v.x / n, v.y / n, v.z / n};
    }
}

Quaternion unit_quaternion(std::mt19937_64& rng) {
    std::normal_distribution<double> g(0.0, 1.0);
    while (true) {
        const Quaternion q{g(rng), g(rng), g(rng), g(rng)};
        if (q.norm() > 1e-6) return q.normalized();
    }
}

void add_c2_track(Scene& s) {
    const Vec3 axis{0.3, 1.0, 0.2};
    const Vec3 trans[5] = {{0, 0, 0}, {0.3, 0.1, 0}, {0, 0.2, 0}, {-0.3, 0.1, 0}, {0, 0, 0}};
    const Vec3 scale[5] = {{1, 1, 1}, {1.3, 0.8, 1.1}, {0.9, 1.2, 0.8}, {1.2, 0.9, 1.3}, {1, 1, 1}};
    AnimationTrack tr;
    tr.object_id = 0;
    for (int k = 0; k < 5; ++k) {
        Keyframe key;
        key.time = k;
        key.rotation = axis_angle_deg(axis, 90.0 * k);
        key.translation = trans[k];
        key.scale = scale[k];
        tr.keys.push_back(key);
    }
    s.objects[0].transform = transform_of(tr.keys.front());
    s.tracks.push_back(tr);
}

void add_c4_instances(Scene& s, const std::shared_ptr<const SvoModel>& model) {
    for (int i = 0; i < 64; ++i) {
        std::mt19937_64 rng(1000 + static_cast<std::uint64_t>(i));
        const Vec3 axis = unit_normal3(rng);
        std::uniform_real_distribution<double> omega_dist(30.0, 120.0), scale_dist(0.6, 1.4);
        const double omega = omega_dist(rng); // degrees per second
        const double s0 = scale_dist(rng);
        const double s1 = scale_dist(rng);
        const double s2 = scale_dist(rng);
        const Vec3 base{((i % 8) - 3.5) * 1.6, ((i / 8) - 3.5) * 1.0, -static_cast<double>((7 * i) % 5)};
        AnimationTrack tr;
        tr.object_id = i;
        for (int k = 0; k <= 16; ++k) {
            const double t = 0.25 * k;
            Keyframe key;
            key.time = t;
            key.rotation = axis_angle_deg(axis, omega * t);
            key.translation = base + Vec3{0.0, 0.2 * std::sin(kPi * t), 0.0};
            const double ph = 2.0 * kPi * t / 1.5;
            key.scale = {s0 * (1.0 + 0.15 * std::sin(ph + 0.0)), s1 * (1.0 + 0.15 * std::sin(ph + 2.0)),
                         s2 * (1.0 + 0.15 * std::sin(ph + 4.0))};
            tr.keys.push_back(key);
        }
        s.objects.push_back(object(i, model, transform_of(tr.keys.front())));
        s.tracks.push_back(tr);
    }
}

void add_crowd(Scene& s, const std::vector<std::shared_ptr<const SvoModel>>& models, int count) {
    for (int i = 0; i < count; ++i) {
        std::mt19937_64 rng(5000 + static_cast<std::uint64_t>(i));
        const Vec3 axis = unit_normal3(rng);
        std::uniform_real_distribution<double> omega_dist(20.0, 90.0), scale_dist(0.5, 0.9);
        const double omega = omega_dist(rng);
        const double sc = scale_dist(rng);
        const Vec3 base{(i % 32) - 15.5, ((i / 32) % 16) - 7.5, -1.5 * (i / 512)};
        AnimationTrack tr;
        tr.object_id = i;
        for (int k = 0; k <= 8; ++k) {
            const double t = 0.5 * k;
            Keyframe key;
            key.time = t;
            key.rotation = axis_angle_deg(axis, omega * t);
            key.translation = base + Vec3{0.0, 0.1 * std::sin(kPi * t + i), 0.0};
            key.scale = {sc, sc, sc};
            tr.keys.push_back(key);
        }
        s.objects.push_back(object(i, models[static_cast<std::size_t>(i) % models.size()], transform_of(tr.keys.front())));
        s.tracks.push_back(tr);
    }
}

} // namespace

Scene make_config_scene(int config, const std::vector<std::shared_ptr<const SvoModel>>& models, std::uint64_t seed,
                        int width, int height) {
    if (models.empty()) throw std::invalid_argument("make_config_scene: no models");
    Scene s;
    int w = 0, h = 0;
    switch (config) {
    case kC1StaticSphere:
        s.objects.push_back(object(0, models[0], RigidTransform{}));
        s.camera = make_look_at_camera({0.3, 0.4, 2.0}, {0, 0, 0}, {0, 1, 0}, 45.0, 512, 512);
        w = 512, h = 512;
        break;
    case kC2Animated:
    case kC3Static:
        s.objects.push_back(object(0, models[0], RigidTransform{}));
        if (config == kC2Animated) add_c2_track(s);
        s.camera = make_look_at_camera({0.0, 0.15, 1.6}, {0, 0, 0}, {0, 1, 0}, 50.0, 1920, 1080);
        w = 1920, h = 1080;
        break;
    case kC4Instances64:
        add_c4_instances(s, models[0]);
        s.camera = make_look_at_camera({0.0, 0.0, 7.5}, {0, 0, -1}, {0, 1, 0}, 60.0, 3840, 2160);
        w = 3840, h = 2160;
        break;
    case kRandomScene: {
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> pos(-3.0, 3.0), scl(0.5, 2.0);
        for (std::size_t i = 0; i < models.size(); ++i) {
            RigidTransform tf;
            tf.translation = {pos(rng), pos(rng), pos(rng)};
            tf.scale = {scl(rng), scl(rng), scl(rng)};
            tf.rotation = rotation_from_quaternion(unit_quaternion(rng));
            s.objects.push_back(object(static_cast<std::int32_t>(i), models[i], tf));
        }
        s.camera = make_look_at_camera({0.0, 0.0, 12.0}, {0, 0, 0}, {0, 1, 0}, 60.0, 160, 120);
        s.background = {10, 20, 30};
        w = 160, h = 120;
        break;
    }
    case kSortedTracing: {
        const Vec3 at[4] = {{6, 0, 0}, {4, 0.75, 0}, {9, 0, 0}, {2, 0.7, 0}};
        for (int i = 0; i < 4; ++i) {
            RigidTransform tf;
            tf.translation = at[i];
            s.objects.push_back(object(i, models[0], tf));
        }
        s.camera = make_look_at_camera({-1, 0.2, 2}, {5, 0.2, 0}, {0, 1, 0}, 70, 64, 48);
        w = 64, h = 48;
        break;
    }
    case kTwoObjects:
    case kHboScene: {
        for (int i = 0; i < 2; ++i) {
            RigidTransform tf;
            tf.translation = {i == 0 ? -2.0 : 2.0, 0, 0};
            tf.scale = {1.5, 1.5, 1.5};
            s.objects.push_back(object(i, models[0], tf));
        }
        if (config == kHboScene) {
            RigidTransform tf;
            tf.translation = {0, 1.5, 1};
            s.objects.push_back(object(2, models.size() > 1 ? models[1] : models[0], tf));
        }
        s.camera = make_look_at_camera({0, 0, 8}, {0, 0, 0}, {0, 1, 0}, 50, 96, 64);
        s.background = {10, 20, 30};
        w = 96, h = 64;
        break;
    }
    case kAxisAligned: {
        s.objects.push_back(object(0, models[0], RigidTransform{}));
        RigidTransform tf;
        tf.translation = {0.75, -0.25, -1.0};
        tf.scale = {0.5, 1.0, 0.75};
        s.objects.push_back(object(1, models.size() > 1 ? models[1] : models[0], tf));
        s.camera = make_look_at_camera({0, 0, 3}, {0, 0, 0}, {0, 1, 0}, 60, 101, 101);
        s.background = {5, 5, 5};
        w = 101, h = 101;
        break;
    }
    case kManyInstances: {
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> jitter(-0.2, 0.2), scl(0.3, 0.6);
        for (int i = 0; i < 200; ++i) {
            RigidTransform tf;
            tf.translation = {(i % 20 - 9.5) * 0.45 + jitter(rng), (i / 20 - 4.5) * 0.45 + jitter(rng),
                              -0.6 * (i % 7) + jitter(rng)};
            tf.scale = {scl(rng), scl(rng), scl(rng)};
            tf.rotation = rotation_from_quaternion(unit_quaternion(rng));
            s.objects.push_back(object(i, models[static_cast<std::size_t>(i) % models.size()], tf));
        }
        s.camera = make_look_at_camera({0, 0, 6}, {0, 0, -1}, {0, 1, 0}, 70, 320, 180);
        w = 320, h = 180;
        break;
    }
    case kCrowd: {
        add_crowd(s, models, seed ? static_cast<int>(seed) : 4096);
        s.camera = make_look_at_camera({0.0, 0.0, 22.0}, {0, 0, 0}, {0, 1, 0}, 60.0, 3840, 2160);
        w = 3840, h = 2160;
        break;
    }
    case kStacked: {
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> jitter(-0.15, 0.15), scl(0.6, 1.2);
        for (int i = 0; i < 96; ++i) {
            RigidTransform tf;
            tf.translation = {jitter(rng), jitter(rng), -0.35 * i};
            tf.scale = {scl(rng), scl(rng), scl(rng)};
            tf.rotation = rotation_from_quaternion(unit_quaternion(rng));
            s.objects.push_back(object(i, models[static_cast<std::size_t>(i) % models.size()], tf));
        }
        s.camera = make_look_at_camera({0, 0, 4}, {0, 0, -1}, {0, 1, 0}, 40, 160, 120);
        w = 160, h = 120;
        break;
    }
    default:
        throw std::invalid_argument("make_config_scene: unknown configuration " + std::to_string(config));
    }
    s.camera.width = width > 0 ? width : w;
    s.camera.height = height > 0 ? height : h;
    return s;
}

} // namespace voxanim::bench
