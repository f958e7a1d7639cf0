// Scene objects, camera and keyframe animation (the per-frame host update).
//
// bounding_sphere: reference proj/src/scene.cpp:16-20. make_look_at_camera:
// scene.cpp:22-55 (columns right, true_up, -forward). evaluate_track:
// scene.cpp:345-368 (clamp, upper_bound segment, lerp a + (b - a) s,
// shortest-arc nlerp). evaluate_animation: scene.cpp:370-385 (dirty iff the
// transform changed exactly). The operand order matches the reference so the
// transforms handed to the GPU are bit-identical to the reference's.
#include "voxanim/scene.hpp"

#include <algorithm>
#include <iterator>
#include <unordered_map>

namespace voxanim {

BoundingSphere bounding_sphere(const SceneObject& object) {
    return {object.transform.translation, 0.5 * object.transform.scale.norm()};
}

Camera make_look_at_camera(const Vec3& position, const Vec3& look_at, const Vec3& up, double vertical_fov_deg,
                           int width, int height) {
    if (!(vertical_fov_deg > 0.0 && vertical_fov_deg < 180.0))
        throw ValidationError("camera fov must be in (0, 180) degrees");
    if (width < 1 || height < 1) throw ValidationError("camera resolution must be at least 1x1");
    const Vec3 view = look_at - position;
    if (view.norm() <= 1e-12) throw ValidationError("camera look_at coincides with its position");
    const Vec3 fwd = view.normalized();
    const Vec3 side = fwd.cross(up);
    if (side.norm() <= 1e-9) throw ValidationError("camera up vector is parallel to the view direction");
    const Vec3 right = side.normalized();
    const Vec3 true_up = right.cross(fwd);
    Camera cam;
    cam.position = position;
    for (int r = 0; r < 3; ++r) {
        cam.orientation(r, 0) = right[r];
        cam.orientation(r, 1) = true_up[r];
        cam.orientation(r, 2) = -fwd[r];
    }
    cam.vertical_fov_deg = vertical_fov_deg;
    cam.width = width;
    cam.height = height;
    cam.dirty = true;
    return cam;
}

SceneObject* Scene::find_object(std::int32_t id) {
    const auto it = std::find_if(objects.begin(), objects.end(), [id](const SceneObject& o) { return o.id == id; });
    return it == objects.end() ? nullptr : &*it;
}

const SceneObject* Scene::find_object(std::int32_t id) const {
    const auto it = std::find_if(objects.begin(), objects.end(), [id](const SceneObject& o) { return o.id == id; });
    return it == objects.end() ? nullptr : &*it;
}

namespace {

// a + (b - a) * s: returns a bitwise when a == b, so constant tracks never
// flip the dirty flag.
double mix(double a, double b, double s) { return a + (b - a) * s; }

Vec3 mix(const Vec3& a, const Vec3& b, double s) { return {mix(a.x, b.x, s), mix(a.y, b.y, s), mix(a.z, b.z, s)}; }

Quaternion nlerp_shortest(const Quaternion& a, Quaternion b, double s) {
    if (a == b) return a;
    if (a.dot(b) < 0.0) {
        b = {-b.w, -b.x, -b.y, -b.z};
        if (a == b) return a;
    }
    return Quaternion{mix(a.w, b.w, s), mix(a.x, b.x, s), mix(a.y, b.y, s), mix(a.z, b.z, s)}.normalized();
}

RigidTransform at_key(const Keyframe& k) {
    RigidTransform tf;
    tf.rotation = rotation_from_quaternion(k.rotation);
    tf.translation = k.translation;
    tf.scale = k.scale;
    return tf;
}

} // namespace

RigidTransform evaluate_track(const AnimationTrack& track, double time) {
    const auto& keys = track.keys;
    if (keys.empty()) throw ValidationError("animation track has no keyframes");
    if (time <= keys.front().time) return at_key(keys.front());
    if (time >= keys.back().time) return at_key(keys.back());
    const auto hi = std::upper_bound(keys.begin(), keys.end(), time,
                                     [](double t, const Keyframe& k) { return t < k.time; });
    const Keyframe& k1 = *hi;
    const Keyframe& k0 = *std::prev(hi);
    const double s = (time - k0.time) / (k1.time - k0.time);
    RigidTransform tf;
    tf.translation = mix(k0.translation, k1.translation, s);
    tf.scale = mix(k0.scale, k1.scale, s);
    tf.rotation = rotation_from_quaternion(nlerp_shortest(k0.rotation, k1.rotation, s));
    return tf;
}

void evaluate_animation(Scene& scene, double time) {
    if (time < 0.0) throw ValidationError("animation time must be nonnegative");
    // The reference resolves each track with Scene::find_object, a linear scan
    // (O(tracks x objects): ~8 M comparisons per frame at 4096 instances). Same
    // answer -- the first object with the id -- from a map built once per call.
    const bool use_map = scene.tracks.size() > 8;
    std::unordered_map<std::int32_t, SceneObject*> by_id;
    if (use_map) {
        by_id.reserve(scene.objects.size());
        for (SceneObject& o : scene.objects) by_id.emplace(o.id, &o); // keeps the first
    }
    for (const AnimationTrack& track : scene.tracks) {
        SceneObject* obj;
        if (use_map) {
            const auto it = by_id.find(track.object_id);
            obj = it == by_id.end() ? nullptr : it->second;
        } else {
            obj = scene.find_object(track.object_id);
        }
        if (obj == nullptr) continue;
        const RigidTransform next = evaluate_track(track, time);
        if (!(next == obj->transform)) {
            obj->transform = next;
            obj->dirty = true;
        }
    }
}

void mark_clean(Scene& scene) {
    for (SceneObject& o : scene.objects) o.dirty = false;
    scene.camera.dirty = false;
}

} // namespace voxanim
