// Benchmark and parity scene definitions (SURVEY.md §8(d) configurations).
//
// Written only against the public voxanim API (scene.hpp / math.hpp), so the
// same source compiles against this library AND against the reference's own
// headers (oracle/Makefile builds it into the reference harness): both sides
// construct bit-identical scenes from the same models, seeds and keyframes.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "voxanim/scene.hpp"

namespace voxanim::bench {

enum SceneConfig : int {
    kC1StaticSphere = 1,   // depth-8 solid sphere, identity, 512x512
    kC2Animated = 2,       // depth-10 shell, rotation+translation+anisotropic scale, 1920x1080
    kC3Static = 3,         // C2 model and camera, identity transform, no animation
    kC4Instances64 = 4,    // 64 animated instances of one depth-11 shell, 3840x2160
    kRandomScene = 5,      // one object per model, seeded random rigid transforms (parity tests)
    kSortedTracing = 6,    // reference test_renderer.cpp:166-179 layout (D, B, A, C along +x)
    kTwoObjects = 7,       // reference test_renderer.cpp:285-293 layout
    kHboScene = 8,         // kTwoObjects + models[1] at (0, 1.5, 1) (test_renderer.cpp:371-374)
    kAxisAligned = 9,      // camera on the z axis, odd resolution: a row and a column of rays with
                           // exactly zero local direction components (zero-direction convention)
    kManyInstances = 10,   // 4 x models.size() x 50 instances on a grid (wide candidate lists)
    kCrowd = 11,           // `seed` (default 4096) animated instances on a 32 x 16 x k lattice, 3840x2160
                           // (scaling with the instance count)
    kStacked = 12,         // 96 instances stacked along the view axis: tile candidate lists
                           // overflow (> 64), exercising the per-ray fallback pass
};

// models: C1-C4 use models[0]; kRandomScene uses every model; kSortedTracing
// and kTwoObjects use models[0] for every object (a full depth-1 cube in the
// reference tests). width/height <= 0 keep the configuration's resolution.
Scene make_config_scene(int config, const std::vector<std::shared_ptr<const SvoModel>>& models, std::uint64_t seed,
                        int width, int height);

// Animation time of frame k in a configuration's sequence (30 fps).
inline double frame_time(int frame) { return frame / 30.0; }

} // namespace voxanim::bench
