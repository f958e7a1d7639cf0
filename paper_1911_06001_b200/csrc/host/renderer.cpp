// Renderer API. render_frame / render_frame_ex hand the whole frame to the
// GPU (vxa_render); the single-ray helpers keep the reference's FP64
// semantics for callers that use them directly:
//   generate_primary_ray  renderer.cpp:11-23
//   ray_sphere_test       renderer.cpp:25-43
//   cull_and_sort         renderer.cpp:45-61 (order (t_center, id))
//   trace_ray             renderer.cpp:63-100 (skip-not-break, nearest (t, id));
//                         each candidate is traversed on the GPU (traverse()).
//   shade                 renderer.cpp:102-113
#include "voxanim/renderer.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <numbers>
#include <thread>
#include <unordered_map>
#include <vector>

#include "voxanim/gpu.hpp"

namespace voxanim {

Ray generate_primary_ray(const Camera& cam, int px, int py) {
    if (px < 0 || py < 0 || px >= cam.width || py >= cam.height)
        throw ValidationError("pixel (" + std::to_string(px) + ", " + std::to_string(py) + ") outside the " +
                              std::to_string(cam.width) + "x" + std::to_string(cam.height) + " image");
    const double tan_half = std::tan(cam.vertical_fov_deg * std::numbers::pi / 360.0);
    const double aspect = static_cast<double>(cam.width) / cam.height;
    const double ndc_x = (px + 0.5) / cam.width * 2.0 - 1.0;
    const double ndc_y = 1.0 - (py + 0.5) / cam.height * 2.0;
    const Vec3 through{ndc_x * tan_half * aspect, ndc_y * tan_half, -1.0};
    return {cam.position, (cam.orientation * through).normalized()};
}

std::optional<SphereHit> ray_sphere_test(const Ray& ray, const BoundingSphere& sphere) {
    const Vec3 l = sphere.center - ray.origin;
    const double tc = l.dot(ray.direction);
    const double d2 = l.norm2() - tc * tc;
    const double r2 = sphere.radius * sphere.radius;
    if (d2 >= r2 || tc + sphere.radius < 0.0) return std::nullopt; // off the line, or entirely behind
    SphereHit h;
    h.d = std::sqrt(std::max(d2, 0.0));
    h.t_center = tc;
    h.t_boundary = std::max(tc - std::sqrt(r2 - d2), 0.0);
    return h;
}

namespace {

bool front_to_back(const SphereHit& a, const SphereHit& b) {
    return a.t_center != b.t_center ? a.t_center < b.t_center : a.object_id < b.object_id;
}

} // namespace

std::vector<SphereHit> cull_and_sort(const Scene& scene, const Ray& ray) {
    std::vector<SphereHit> out;
    out.reserve(scene.objects.size());
    for (const SceneObject& o : scene.objects) {
        if (auto h = ray_sphere_test(ray, bounding_sphere(o))) {
            h->object_id = o.id;
            out.push_back(*h);
        }
    }
    std::sort(out.begin(), out.end(), front_to_back);
    return out;
}

HitRecord trace_ray(const Scene& scene, const Ray& ray, std::span<const SphereHit> candidates, FrameStats* stats) {
    HitRecord best;
    bool have = false;
    for (const SphereHit& c : candidates) {
        if (have && best.t < c.t_boundary) continue; // nothing inside this sphere can be nearer
        const SceneObject* obj = scene.find_object(c.object_id);
        if (obj == nullptr || !obj->model) continue;
        const Ray local = transform_ray_world_to_local(ray, obj->transform);
        if (stats) ++stats->svo_traversals;
        const auto hit = traverse(*obj->model, local, bounds_from_scale(obj->transform.scale));
        if (!hit) continue;
        if (!have || hit->t_hit < best.t || (hit->t_hit == best.t && obj->id < best.object_id)) {
            have = true;
            best.color = hit->attribute;
            best.normal = obj->transform.rotation * hit->normal_local;
            best.t = hit->t_hit;
            best.object_id = obj->id;
        }
    }
    if (have) best.kind = candidates.size() > 1 ? HitKind::MultiSphere : HitKind::SingleSphere;
    return best;
}

std::array<std::uint8_t, 3> shade(const HitRecord& rec, const Ray& ray, const std::array<std::uint8_t, 3>& background) {
    if (rec.kind == HitKind::Miss) return background;
    const double f = 0.2 + 0.8 * std::max(0.0, rec.normal.dot(-ray.direction));
    const auto q = [f](std::uint8_t c) { return static_cast<std::uint8_t>(std::lround(c * f)); };
    return {q(rec.color.r), q(rec.color.g), q(rec.color.b)};
}

// ---- HitBuffer: GPU-resident, host copy synced on access
HitBuffer::HitBuffer(int width, int height)
    : w_(width), h_(height), rec_(static_cast<std::size_t>(width) * static_cast<std::size_t>(height)),
      mu_(std::make_unique<std::mutex>()) {}

HitBuffer::HitBuffer(const HitBuffer& other)
    : w_(other.w_), h_(other.h_), rec_((other.sync_host(), other.rec_)), host_newer_(true),
      mu_(std::make_unique<std::mutex>()) {}

HitBuffer::HitBuffer(HitBuffer&& other) noexcept
    : w_(other.w_), h_(other.h_), rec_(std::move(other.rec_)), dev_(other.dev_),
      gpu_newer_(other.gpu_newer_.load()), host_newer_(other.host_newer_), mu_(std::make_unique<std::mutex>()) {
    other.dev_ = 0;
    other.gpu_newer_ = false;
}

HitBuffer& HitBuffer::operator=(const HitBuffer& other) {
    if (this != &other) {
        other.sync_host();
        release_device();
        w_ = other.w_;
        h_ = other.h_;
        rec_ = other.rec_;
        gpu_newer_ = false;
        host_newer_ = true;
    }
    return *this;
}

HitBuffer& HitBuffer::operator=(HitBuffer&& other) noexcept {
    if (this != &other) {
        release_device();
        w_ = other.w_;
        h_ = other.h_;
        rec_ = std::move(other.rec_);
        dev_ = other.dev_;
        gpu_newer_ = other.gpu_newer_.load();
        host_newer_ = other.host_newer_;
        other.dev_ = 0;
        other.gpu_newer_ = false;
    }
    return *this;
}

HitBuffer::~HitBuffer() { release_device(); }

void HitBuffer::release_device() noexcept {
    if (dev_ != 0) {
        try {
            vxa_hbo_release(gpu::context(), dev_);
        } catch (...) {
        }
        dev_ = 0;
    }
}

void HitBuffer::pull() const {
    std::lock_guard<std::mutex> lk(*mu_);
    if (!gpu_newer_.load(std::memory_order_relaxed)) return;
    gpu::check(vxa_hbo_download(gpu::context(), dev_, reinterpret_cast<vxa_hit_record*>(rec_.data())),
               "vxa_hbo_download");
    gpu_newer_.store(false, std::memory_order_release);
}

std::uint32_t HitBuffer::device_for_frame() {
    vxa_ctx* ctx = gpu::context();
    if (dev_ == 0) {
        gpu::check(vxa_hbo_create(ctx, w_, h_, &dev_), "vxa_hbo_create"); // Miss records, like a fresh buffer
    }
    if (host_newer_) {
        sync_host();
        gpu::check(vxa_hbo_upload(ctx, dev_, reinterpret_cast<const vxa_hit_record*>(rec_.data())), "vxa_hbo_upload");
        host_newer_ = false;
    }
    return dev_;
}

namespace gpu {

void render_frame_into(const Scene& scene, const RenderOptions& opts, const RenderOptionsEx& ex, FrameStats& stats,
                       std::uint8_t* rgb_out, vxa_stats* device_stats) {
    const Camera& cam = scene.camera;
    if (opts.hbo && (opts.hbo->width() != cam.width || opts.hbo->height() != cam.height))
        throw ValidationError("hit buffer dimensions do not match the camera");
    const auto t0 = std::chrono::steady_clock::now();

    std::vector<vxa_instance> inst(scene.objects.size());
    std::unordered_map<const SvoModel*, std::uint32_t> handles;
    begin_model_frame();
    for (std::size_t i = 0; i < scene.objects.size(); ++i) {
        const SceneObject& o = scene.objects[i];
        vxa_instance& v = inst[i];
        v = vxa_instance{};
        v.id = o.id;
        if (o.model) {
            auto [it, fresh] = handles.try_emplace(o.model.get(), 0u);
            if (fresh) it->second = model_handle(o.model);
            v.model = it->second;
        }
        std::copy(o.transform.rotation.m.begin(), o.transform.rotation.m.end(), v.rotation);
        for (int k = 0; k < 3; ++k) {
            v.translation[k] = o.transform.translation[k];
            v.scale[k] = o.transform.scale[k];
        }
        v.dirty = o.dirty ? 1 : 0;
    }

    vxa_frame_desc f{};
    for (int k = 0; k < 3; ++k) f.camera.position[k] = cam.position[k];
    std::copy(cam.orientation.m.begin(), cam.orientation.m.end(), f.camera.orientation);
    f.camera.vertical_fov_deg = cam.vertical_fov_deg;
    f.camera.width = cam.width;
    f.camera.height = cam.height;
    f.background[0] = scene.background[0];
    f.background[1] = scene.background[1];
    f.background[2] = scene.background[2];
    f.culling = opts.culling ? 1 : 0;
    f.sorting = opts.sorting ? 1 : 0;
    f.precision = static_cast<std::uint8_t>(ex.precision);
    f.camera_dirty = cam.dirty ? 1 : 0;
    f.tile_rank = ex.tile_rank;
    f.tile_world = ex.tile_world;
    f.hbo = nullptr;
    f.hbo_device = opts.hbo ? opts.hbo->device_for_frame() : 0; // GPU-resident, no per-frame transfers

    if (ex.aov) ex.aov->resize(static_cast<std::size_t>(cam.width) * static_cast<std::size_t>(cam.height));
    vxa_stats ds{};
    check(vxa_render(context(), &f, inst.data(), static_cast<std::uint32_t>(inst.size()),
                     rgb_out, ex.aov ? ex.aov->data() : nullptr, &ds),
          "vxa_render");
    if (opts.hbo) opts.hbo->frame_written();
    stats = FrameStats{};
    stats.rays = ds.rays;
    stats.sphere_tests = ds.sphere_tests;
    stats.svo_traversals = ds.svo_traversals;
    stats.pixels_reused = ds.pixels_reused;
    stats.render_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (device_stats) *device_stats = ds;
}

namespace {
// render_frame returns its Image by value (renderer.hpp:126): a fresh, zero-filled,
// pageable vector every call. Rendering straight into it would take the banded
// pageable copies, and the zero fill alone costs about a frame's kernel time. So
// the frame is rendered into a page-locked staging image (the direct readback:
// the frame kernel stores each finished super-tile into it over PCIe) while a
// worker builds the Image, and the staging image is then copied into the Image by
// a few threads.
class ImageStaging {
public:
    static ImageStaging& get() {
        static ImageStaging s;
        return s;
    }
    std::mutex mu; // one render_frame at a time uses the staging image

    // staging image of at least n bytes, page-locked for the context (grow-only)
    uint8_t* ensure(size_t n) {
        if (n <= cap_) return buf_;
        if (buf_) {
            vxa_host_unregister(context(), buf_);
            std::free(buf_);
            buf_ = nullptr;
            cap_ = 0;
        }
        const size_t bytes = (n + 4095) & ~size_t{4095};
        void* p = std::aligned_alloc(4096, bytes);
        if (p == nullptr) return nullptr;
        if (vxa_host_register(context(), p, bytes) != VXA_OK) {
            std::free(p);
            return nullptr;
        }
        buf_ = static_cast<uint8_t*>(p);
        cap_ = bytes;
        return buf_;
    }

    // f() on a worker; wait() joins it
    void run_async(std::function<void()> f) { submit({std::move(f)}); }
    void wait() { wait_all(); }

    // dst[0, n) = src[0, n) in chunks over the workers and the calling thread
    void parallel_copy(uint8_t* dst, const uint8_t* src, size_t n) {
        const size_t parts = workers_.size() + 1;
        const size_t chunk = ((n + parts - 1) / parts + 63) & ~size_t{63};
        std::vector<std::function<void()>> jobs;
        for (size_t k = 1; k < parts; ++k) {
            const size_t a = std::min(n, k * chunk), b = std::min(n, a + chunk);
            if (a < b) jobs.emplace_back([=] { std::memcpy(dst + a, src + a, b - a); });
        }
        submit(std::move(jobs));
        std::memcpy(dst, src, std::min(n, chunk));
        wait_all();
    }

private:
    ImageStaging() {
        const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
        const unsigned n = std::min(8u, hw - 1);
        for (unsigned k = 0; k < n; ++k) workers_.emplace_back([this] { loop(); });
    }
    ~ImageStaging() {
        {
            std::lock_guard<std::mutex> lk(q_mu_);
            stop_ = true;
        }
        q_cv_.notify_all();
        for (auto& t : workers_) t.join();
        // the staging image stays registered until the process ends (the context may be gone)
    }
    void submit(std::vector<std::function<void()>> jobs) {
        {
            std::lock_guard<std::mutex> lk(q_mu_);
            for (auto& j : jobs) queue_.push_back(std::move(j));
            pending_ += jobs.size();
        }
        q_cv_.notify_all();
    }
    void wait_all() {
        std::unique_lock<std::mutex> lk(q_mu_);
        done_cv_.wait(lk, [this] { return pending_ == 0; });
    }
    void loop() {
        while (true) {
            std::function<void()> job;
            {
                std::unique_lock<std::mutex> lk(q_mu_);
                q_cv_.wait(lk, [this] { return stop_ || !queue_.empty(); });
                if (stop_ && queue_.empty()) return;
                job = std::move(queue_.back());
                queue_.pop_back();
            }
            job();
            {
                std::lock_guard<std::mutex> lk(q_mu_);
                if (--pending_ == 0) done_cv_.notify_all();
            }
        }
    }
    uint8_t* buf_ = nullptr;
    size_t cap_ = 0;
    std::vector<std::thread> workers_;
    std::mutex q_mu_;
    std::condition_variable q_cv_, done_cv_;
    std::vector<std::function<void()>> queue_;
    size_t pending_ = 0;
    bool stop_ = false;
};

// Images built ahead: two threads keep up to two zero-filled Images of the last
// frame size ready, so the constructor's zero fill (2.6 ms at 4K on the GPU box,
// single-threaded) runs beside the callers' frames instead of inside them.
// VOXANIM_IMAGE_SPARES=0 turns it off.
class SpareImages {
public:
    static SpareImages& get() {
        static SpareImages s;
        return s;
    }
    // an Image of w x h: a ready one, one being built, or a new one
    Image take(int w, int h) {
        std::unique_lock<std::mutex> lk(mu_);
        if (w != w_ || h != h_) {
            w_ = w, h_ = h;
            ready_.clear();
            cv_.notify_all();
        }
        if (ready_.empty() && building_ > 0) cv_.wait(lk, [&] { return !ready_.empty() || building_ == 0; });
        if (!ready_.empty()) {
            Image img = std::move(ready_.back());
            ready_.pop_back();
            cv_.notify_all(); // a builder refills
            return img;
        }
        lk.unlock();
        return Image(w, h);
    }

private:
    static constexpr size_t kTarget = 2;
    SpareImages() {
        for (size_t k = 0; k < kTarget; ++k) th_.emplace_back([this] { build_loop(); });
    }
    ~SpareImages() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void build_loop() {
        std::unique_lock<std::mutex> lk(mu_);
        while (true) {
            cv_.wait(lk, [&] { return stop_ || (w_ > 0 && ready_.size() + building_ < kTarget); });
            if (stop_) return;
            const int w = w_, h = h_;
            ++building_;
            lk.unlock();
            Image img(w, h);
            lk.lock();
            --building_;
            if (w == w_ && h == h_) ready_.push_back(std::move(img));
            cv_.notify_all();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    int w_ = 0, h_ = 0;
    std::vector<Image> ready_;
    size_t building_ = 0;
    bool stop_ = false;
    std::vector<std::thread> th_;
};
} // namespace

Image render_frame_ex(const Scene& scene, const RenderOptions& opts, const RenderOptionsEx& ex, FrameStats& stats,
                      vxa_stats* device_stats) {
    Image image;
    const int w = scene.camera.width, h = scene.camera.height;
    const size_t n = static_cast<size_t>(w) * static_cast<size_t>(h) * 3;
    const char* env = std::getenv("VOXANIM_IMAGE_STAGING");
    const bool staged = ex.read_image && ex.aov == nullptr && n >= (size_t{3} << 20) &&
                        !(env && std::strcmp(env, "0") == 0);
    if (staged) {
        ImageStaging& st = ImageStaging::get();
        std::unique_lock<std::mutex> lk(st.mu);
        if (uint8_t* stage = st.ensure(n)) {
            // the Image (allocation + zero fill) is built while the GPU renders, or
            // taken ready from the spares
            const char* sp = std::getenv("VOXANIM_IMAGE_SPARES");
            const bool spares = !(sp && std::strcmp(sp, "0") == 0);
            st.run_async([&image, w, h, spares] { image = spares ? SpareImages::get().take(w, h) : Image(w, h); });
            try {
                render_frame_into(scene, opts, ex, stats, stage, device_stats);
            } catch (...) {
                st.wait();
                throw;
            }
            st.wait();
            st.parallel_copy(image.rgb.data(), stage, n);
            return image;
        }
    }
    if (ex.read_image) image = Image(w, h);
    render_frame_into(scene, opts, ex, stats, ex.read_image ? image.rgb.data() : nullptr, device_stats);
    return image;
}

} // namespace gpu

Image render_frame(const Scene& scene, const RenderOptions& opts, FrameStats& stats) {
    gpu::RenderOptionsEx ex;
    ex.precision = gpu::default_precision();
    return gpu::render_frame_ex(scene, opts, ex, stats);
}

std::string write_ppm(const Image& image) {
    std::string out = "P6\n" + std::to_string(image.width) + " " + std::to_string(image.height) + "\n255\n";
    out.append(reinterpret_cast<const char*>(image.rgb.data()), image.rgb.size());
    return out;
}

} // namespace voxanim
