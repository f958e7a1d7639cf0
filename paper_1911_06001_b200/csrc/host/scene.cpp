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
#include <cmath>
#include <fstream>
#include <iterator>
#include <map>
#include <numbers>
#include <sstream>
#include <unordered_map>

#include "json_lite.hpp"

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

// ---------------------------------------------------------------------------
// Scene documents (reference scene.cpp:75-306): the same schema, the same
// check order and error texts, over this library's own JSON reader.

namespace {

using json_lite::Value;

Vec3 vec3_of(const Value& j, const std::string& where) {
    if (!j.is_array() || j.size() != 3 || !j[0].is_number() || !j[1].is_number() || !j[2].is_number())
        throw ParseError("scene: " + where + " must be an array of 3 numbers");
    return {j[0].number(), j[1].number(), j[2].number()};
}

double number_of(const Value& j, const std::string& where) {
    if (!j.is_number()) throw ParseError("scene: " + where + " must be a number");
    return j.number();
}

// {"quat": [w, x, y, z]} (normalised) or {"axis": [x, y, z], "angle_deg": a}
Quaternion rotation_of(const Value& j, const std::string& where) {
    if (j.contains("quat")) {
        const Value& q = j["quat"];
        if (!q.is_array() || q.size() != 4) throw ParseError("scene: " + where + ".quat must be an array of 4 numbers");
        const Quaternion quat{number_of(q[0], where + ".quat[0]"), number_of(q[1], where + ".quat[1]"),
                              number_of(q[2], where + ".quat[2]"), number_of(q[3], where + ".quat[3]")};
        if (quat.norm() <= 1e-12) throw ValidationError("scene: bad rotation at " + where + " (near-zero quaternion)");
        return quat.normalized();
    }
    if (j.contains("axis")) {
        const Vec3 axis = vec3_of(j["axis"], where + ".axis");
        if (!j.contains("angle_deg") || !j["angle_deg"].is_number())
            throw ParseError("scene: " + where + " needs a numeric angle_deg");
        if (axis.norm() <= 1e-12) throw ValidationError("scene: bad rotation at " + where + " (near-zero axis)");
        return Quaternion::from_axis_angle(axis, j["angle_deg"].number() * std::numbers::pi / 180.0);
    }
    throw ParseError("scene: " + where + " must contain either quat or axis/angle_deg");
}

void require_positive(const Vec3& scale, const std::string& where) {
    if (!(scale.x > 0.0 && scale.y > 0.0 && scale.z > 0.0))
        throw ValidationError("scene: " + where + " scale components must be positive");
}

std::int32_t int32_of(const Value& j) { return static_cast<std::int32_t>(j.integer()); }

void load_models(const Value& doc, const std::filesystem::path& base_dir,
                 std::map<std::string, std::shared_ptr<const SvoModel>>& models) {
    if (!doc.contains("models")) return;
    const Value& m = doc["models"];
    if (!m.is_object()) throw ParseError("scene: models must map names to paths");
    for (const auto& [name, value] : m.o) { // key order
        if (!value.is_string()) throw ParseError("scene: models." + name + " must be a path string");
        const std::filesystem::path path = base_dir / value.s;
        if (!std::filesystem::exists(path))
            throw IoError("scene: model not found: " + path.string() + " (models." + name + ")");
        auto model = std::make_shared<SvoModel>(load_svo(path));
        if (const SvoValidationReport rep = validate(*model); !rep.ok())
            throw ValidationError("scene: model " + name + " fails validation: " + rep.violations.front().message);
        models.emplace(name, std::move(model));
    }
}

void load_objects(const Value& doc, const std::map<std::string, std::shared_ptr<const SvoModel>>& models, Scene& scene) {
    if (!doc.contains("objects")) return;
    const Value& list = doc["objects"];
    if (!list.is_array()) throw ParseError("scene: objects must be an array");
    for (std::size_t k = 0; k < list.a.size(); ++k) {
        const Value& j = list.a[k];
        const std::string where = "objects[" + std::to_string(k) + "]";
        SceneObject obj;
        if (!j.contains("id") || !j["id"].is_number_integer()) throw ParseError("scene: " + where + " needs an integer id");
        obj.id = int32_of(j["id"]);
        if (scene.find_object(obj.id))
            throw ValidationError("scene: duplicate object id " + std::to_string(obj.id) + " at " + where);
        if (!j.contains("model") || !j["model"].is_string()) throw ParseError("scene: " + where + " needs a model name");
        obj.model_name = j["model"].s;
        const auto it = models.find(obj.model_name);
        if (it == models.end())
            throw ValidationError("scene: " + where + " references unknown model \"" + obj.model_name + "\"");
        obj.model = it->second;
        if (j.contains("translation")) obj.transform.translation = vec3_of(j["translation"], where + ".translation");
        if (j.contains("rotation"))
            obj.transform.rotation = rotation_from_quaternion(rotation_of(j["rotation"], where + ".rotation"));
        if (j.contains("scale")) obj.transform.scale = vec3_of(j["scale"], where + ".scale");
        require_positive(obj.transform.scale, where);
        obj.dirty = false;
        scene.objects.push_back(std::move(obj));
    }
}

void load_tracks(const Value& doc, Scene& scene) {
    if (!doc.contains("tracks")) return;
    const Value& list = doc["tracks"];
    if (!list.is_array()) throw ParseError("scene: tracks must be an array");
    for (std::size_t k = 0; k < list.a.size(); ++k) {
        const Value& j = list.a[k];
        const std::string where = "tracks[" + std::to_string(k) + "]";
        AnimationTrack track;
        if (!j.contains("object") || !j["object"].is_number_integer())
            throw ParseError("scene: " + where + " needs an integer object id");
        track.object_id = int32_of(j["object"]);
        if (!scene.find_object(track.object_id))
            throw ValidationError("scene: " + where + " references unknown object id " + std::to_string(track.object_id));
        if (!j.contains("keys") || !j["keys"].is_array() || j["keys"].a.empty())
            throw ParseError("scene: " + where + " needs a nonempty keys array");
        const Value& keys = j["keys"];
        for (std::size_t q = 0; q < keys.a.size(); ++q) {
            const Value& kj = keys.a[q];
            const std::string kw = where + ".keys[" + std::to_string(q) + "]";
            Keyframe key;
            if (!kj.contains("time") || !kj["time"].is_number()) throw ParseError("scene: " + kw + " needs a numeric time");
            key.time = kj["time"].number();
            if (kj.contains("translation")) key.translation = vec3_of(kj["translation"], kw + ".translation");
            if (kj.contains("rotation")) key.rotation = rotation_of(kj["rotation"], kw + ".rotation");
            if (kj.contains("scale")) key.scale = vec3_of(kj["scale"], kw + ".scale");
            require_positive(key.scale, kw);
            if (!track.keys.empty() && key.time <= track.keys.back().time)
                throw ValidationError("scene: " + kw + " keyframe times must be strictly increasing");
            track.keys.push_back(key);
        }
        scene.tracks.push_back(std::move(track));
    }
}

} // namespace

Scene load_scene(const std::string& text, const std::filesystem::path& base_dir) {
    Value doc;
    try {
        doc = json_lite::parse(text);
    } catch (const json_lite::Error& e) {
        throw ParseError(std::string("scene: invalid JSON: ") + e.what());
    }
    if (!doc.is_object()) throw ParseError("scene: top level must be an object");

    Scene scene;
    std::map<std::string, std::shared_ptr<const SvoModel>> models;
    load_models(doc, base_dir, models);
    load_objects(doc, models, scene);
    load_tracks(doc, scene);

    // camera: defaults at the origin looking down -z, fov 60, 640x480
    Vec3 position{0, 0, 0}, look_at{0, 0, -1}, up{0, 1, 0};
    double fov = 60.0;
    if (doc.contains("camera")) {
        const Value& c = doc["camera"];
        if (!c.is_object()) throw ParseError("scene: camera must be an object");
        if (c.contains("position")) position = vec3_of(c["position"], "camera.position");
        if (c.contains("look_at")) look_at = vec3_of(c["look_at"], "camera.look_at");
        if (c.contains("up")) up = vec3_of(c["up"], "camera.up");
        if (c.contains("fov_deg")) {
            if (!c["fov_deg"].is_number()) throw ParseError("scene: camera.fov_deg must be a number");
            fov = c["fov_deg"].number();
        }
    }
    scene.camera = make_look_at_camera(position, look_at, up, fov, 640, 480);

    if (doc.contains("background")) {
        const Value& b = doc["background"];
        if (!b.is_array() || b.size() != 3)
            throw ParseError("scene: background must be an array of 3 numbers (0..255)");
        for (std::size_t k = 0; k < 3; ++k) {
            const double v = number_of(b[k], "background[" + std::to_string(k) + "]");
            if (v < 0.0 || v > 255.0) throw ValidationError("scene: background channels must be in [0, 255]");
            scene.background[k] = static_cast<std::uint8_t>(std::lround(v));
        }
    }
    return scene;
}

Scene load_scene_file(const std::filesystem::path& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open scene: " + path.string());
    std::ostringstream text;
    text << in.rdbuf();
    return load_scene(text.str(), path.has_parent_path() ? path.parent_path() : std::filesystem::path("."));
}

} // namespace voxanim
