/*
 * voxanim_capi.h — flat C binding of the voxanim C++ API (libvoxanim.so).
 *
 * This is the "ctypes stub" layer: it lets Python (tests, bench.py) drive
 * the same calls a C++ user of the reference makes — build/load a model,
 * build a scene, evaluate_animation, render_frame — without touching C++
 * types. Handles own C++ objects (shared_ptr<const SvoModel>, Scene,
 * HitBuffer). All functions return 0 / a handle on success and a negative
 * value / NULL on failure with vxn_last_error() set.
 */
#ifndef VOXANIM_CAPI_H
#define VOXANIM_CAPI_H

#include <stddef.h>
#include <stdint.h>

#include "vxa.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vxn_model vxn_model;
typedef struct vxn_scene vxn_scene;
typedef struct vxn_hbo vxn_hbo;

const char* vxn_last_error(void);

/* models */
vxn_model* vxn_model_procedural(int shell, uint32_t depth);      /* sparse builder, any depth <= 16 */
vxn_model* vxn_model_dense_sphere(uint32_t depth);               /* build_from_grid(gen_primitive(Sphere)) */
vxn_model* vxn_model_random(uint64_t seed, uint32_t depth, double fill); /* mt19937_64 random grid */
vxn_model* vxn_model_full_cube(void);                            /* depth-1 model, all 8 voxels */
/* build_from_grid of a dense VoxelGrid bitset ((n^3+63)/64 words, n = 2^depth, x-major)
 * with ColorSpec{color_mode, color_rgba}; device != 0 builds it on the GPU (vxa_build_model). */
vxn_model* vxn_model_from_grid(const uint64_t* words, uint32_t depth, uint32_t color_mode, uint32_t color_rgba,
                               int device);
/* gen_primitive(kind, depth) bitset (kind: 0 Sphere, 1 BoxShell, 2 Menger, 3 Checker) into out
 * (cap_words words; out may be NULL to query); *grid_depth = log2 of its resolution (Menger:
 * 3^depth rounded up to a power of two). Returns the word count, or -1. */
int64_t vxn_grid_primitive(int kind, uint32_t depth, uint64_t* out, size_t cap_words, uint32_t* grid_depth);
vxn_model* vxn_model_deserialize(const uint8_t* bytes, size_t n);
int vxn_model_save(const vxn_model* m, const char* path);         /* save_svo */
int64_t vxn_model_serialize(const vxn_model* m, uint8_t* out, size_t cap); /* returns the size */
int vxn_model_info(const vxn_model* m, uint32_t* depth, uint64_t* nodes, uint64_t* attrs);
int vxn_model_validate(const vxn_model* m);                     /* number of violations */
void vxn_model_free(vxn_model* m);

/* scenes (bench_scenes.hpp configurations) */
/* load_scene_file(path) with the camera resolution set to width x height (the CLI's bench) */
vxn_scene* vxn_scene_load(const char* path, int width, int height);
vxn_scene* vxn_scene_config(int config, vxn_model* const* models, uint32_t n_models, uint64_t seed, int width,
                            int height);
int vxn_scene_evaluate(vxn_scene* s, double time);
int vxn_scene_mark_clean(vxn_scene* s);
int vxn_scene_set_camera_dirty(vxn_scene* s, int dirty);
/* camera = make_look_at_camera(position, look_at, up, fov, width, height) (scene.cpp:22-55); dirty set */
int vxn_scene_set_camera(vxn_scene* s, const double* position3, const double* look_at3, const double* up3,
                         double vertical_fov_deg, int width, int height);
int vxn_scene_object_count(const vxn_scene* s);
/* Per-object RigidTransform (15 doubles: rotation 9, translation 3, scale 3) + dirty flag. */
int vxn_scene_get_object(const vxn_scene* s, int index, int32_t* id, double* transform15, int* dirty);
int vxn_scene_set_object(vxn_scene* s, int index, const double* transform15, int dirty);
/* The C-ABI view of the scene: frame descriptor (camera, background) and
 * instances with model handles on the library's global context. */
int vxn_scene_export(vxn_scene* s, vxa_frame_desc* frame, vxa_instance* instances, uint32_t cap, uint32_t* count);
void vxn_scene_free(vxn_scene* s);

/* One benchmark step without Python in the loop, the reference bench loop
 * (cli.cpp:265-270): evaluate_animation(time) (skipped when time < 0), build
 * the instance table, vxa_submit the frame (precision, screen-tile
 * rank/world, optional device hit buffer) on the global context, mark_clean. */
int vxn_scene_submit(vxn_scene* s, double time, int precision, int rank, int world, uint32_t hbo_device);

/* Streaming step: evaluate_animation(time), frame + asynchronous RGB8 readback
 * into rgb_out (vxa_submit_readback); wait with vxa_wait_readback(ticket). */
int vxn_scene_stream(vxn_scene* s, double time, int precision, uint8_t* rgb_out, uint64_t* ticket);

vxn_hbo* vxn_hbo_create(int width, int height);
void vxn_hbo_free(vxn_hbo* h);
/* HitBuffer records through its host accessors (width*height 48-byte records) */
int vxn_hbo_records(vxn_hbo* h, vxa_hit_record* out);
int vxn_hbo_set_record(vxn_hbo* h, int x, int y, const vxa_hit_record* rec);

/* voxanim::render_frame (precision < 0: library default) / render_frame_ex.
 * rgb: width*height*3 or NULL (frame stays on the device); aov: width*height
 * records or NULL; fs: FrameStats {rays, sphere_tests, svo_traversals,
 * pixels_reused} as 4 uint64 + render_ms; ds: device stats (may be NULL). */
int vxn_render(vxn_scene* s, int culling, int sorting, int precision, vxn_hbo* hbo, uint8_t* rgb,
               vxa_pixel_aov* aov, uint64_t* fs4, double* render_ms, vxa_stats* ds);

/* The drop-in voxanim::render_frame (Image returned by value) `steps` times at
 * animation times time + k/30: mean wall time per call (ms_per_call) and the
 * last image's RGB8 bytes copied to last_rgb (width*height*3, or NULL). */
int vxn_scene_render_image(vxn_scene* s, double time, int steps, double* ms_per_call, uint8_t* last_rgb);

/* voxanim::traverse on a batch of local rays (vxa_local_ray), FP64, through
 * the C++ API (which dispatches to vxa_traverse). */
int vxn_traverse(const vxn_model* m, const vxa_local_ray* rays, uint32_t n, vxa_traverse_hit* hits);

/* The process-wide context render_frame uses (for timers / L2 flush). */
vxa_ctx* vxn_context(void);

#ifdef __cplusplus
}
#endif

#endif
