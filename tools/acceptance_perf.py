"""The reference's own performance criteria (proj/tests/acceptance/acceptance.cpp,
criteria 5 and 6) measured on the GPU path through the drop-in
API: the acceptance fixture (the same four primitive models, scene documents
and bench configurations) is rebuilt with this library (build_from_grid,
save_svo, load_scene_file) and run in the reference CLI's bench modes.

  5. animated-opt <= 0.9 x animated   (bench scene: 4 objects, 2 animated, 640x480, 60 frames)
  6. animated     <= 1.4 x static     (single scene: 1 slowly rotating object, 320x240, 40 frames)
  7. fps * avg_ms = 1000 +- 0.1 %      (report consistency)

    python tools/acceptance_perf.py        # prints one JSON object
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from voxanim_bench import run_mode  # noqa: E402

# acceptance.cpp:54-96, verbatim scene documents
BENCH_SCENE = """{
  "models": {"menger": "menger.svo", "shell": "shell.svo", "ball": "ball.svo", "check": "check.svo"},
  "objects": [
    {"id": 0, "model": "menger", "translation": [-4.5, 0, 0], "scale": [2, 2, 2]},
    {"id": 1, "model": "shell",  "translation": [4.5, 0, 0],  "scale": [2, 2, 2]},
    {"id": 2, "model": "ball",   "translation": [-1.8, 1.6, 0], "scale": [1.2, 1.2, 1.2]},
    {"id": 3, "model": "check",  "translation": [1.4, -1.6, 0], "scale": [1.2, 1.2, 1.2]}
  ],
  "tracks": [
    {"object": 2, "keys": [
      {"time": 0, "translation": [-1.8, 1.6, 0], "scale": [1.2, 1.2, 1.2]},
      {"time": 1, "translation": [-1.0, 1.6, 0], "scale": [1.2, 1.2, 1.2]},
      {"time": 2, "translation": [-1.8, 1.6, 0], "scale": [1.2, 1.2, 1.2]}
    ]},
    {"object": 3, "keys": [
      {"time": 0, "rotation": {"axis": [0, 1, 0], "angle_deg": 0}, "translation": [1.4, -1.6, 0], "scale": [1.2, 1.2, 1.2]},
      {"time": 1, "rotation": {"axis": [0, 1, 0], "angle_deg": 90}, "translation": [1.4, -1.6, 0], "scale": [1.2, 1.2, 1.2]},
      {"time": 2, "rotation": {"axis": [0, 1, 0], "angle_deg": 180}, "translation": [1.4, -1.6, 0], "scale": [1.2, 1.2, 1.2]}
    ]}
  ],
  "camera": {"position": [0, 0.4, 11], "look_at": [0, 0, 0], "fov_deg": 55},
  "background": [12, 14, 26]
}"""
SINGLE_SCENE = """{
  "models": {"menger": "menger.svo"},
  "objects": [{"id": 0, "model": "menger", "scale": [2.5, 2.5, 2.5]}],
  "tracks": [{"object": 0, "keys": [
    {"time": 0, "rotation": {"axis": [0, 1, 0], "angle_deg": 0},  "scale": [2.5, 2.5, 2.5]},
    {"time": 4, "rotation": {"axis": [0, 1, 0], "angle_deg": 40}, "scale": [2.5, 2.5, 2.5]}
  ]}],
  "camera": {"position": [0, 1.5, 6.5], "look_at": [0, 0, 0], "fov_deg": 60}
}"""


def build_fixture(vx, d: str) -> None:
    # acceptance.cpp:46-53: cmd_build(shape, depth) = build_from_grid(gen_primitive(shape, depth))
    for shape, depth, name in (("menger", 3, "menger.svo"), ("box_shell", 4, "shell.svo"),
                               ("sphere", 4, "ball.svo"), ("checker", 3, "check.svo")):
        words, grid_depth = vx.grid_primitive(shape, depth)
        vx.Model.from_grid(words, grid_depth, device=False).save(os.path.join(d, name))
    with open(os.path.join(d, "bench.json"), "w") as f:
        f.write(BENCH_SCENE)
    with open(os.path.join(d, "single.json"), "w") as f:
        f.write(SINGLE_SCENE)


def avg(ms):
    return sum(ms) / len(ms)


def measure() -> dict:
    import paper_1911_06001_b200 as vx

    with tempfile.TemporaryDirectory(prefix="voxanim_acceptance_") as d:
        build_fixture(vx, d)
        bench = os.path.join(d, "bench.json")
        single = os.path.join(d, "single.json")
        anim, _ = run_mode(vx, vx.Scene.load(bench, 640, 480), "animated", 60, 30.0, 640, 480)
        opt, _ = run_mode(vx, vx.Scene.load(bench, 640, 480), "animated-opt", 60, 30.0, 640, 480)
        stat, _ = run_mode(vx, vx.Scene.load(single, 320, 240), "static", 40, 30.0, 320, 240)
        anim1, _ = run_mode(vx, vx.Scene.load(single, 320, 240), "animated", 40, 30.0, 320, 240)
    out = {
        "criterion_5": {"animated_ms": round(avg(anim), 4), "animated_opt_ms": round(avg(opt), 4),
                        "ratio": round(avg(opt) / avg(anim), 4), "threshold": 0.9,
                        "ok": avg(opt) <= 0.9 * avg(anim)},
        "criterion_6": {"static_ms": round(avg(stat), 4), "animated_ms": round(avg(anim1), 4),
                        "ratio": round(avg(anim1) / avg(stat), 4), "threshold": 1.4,
                        "ok": avg(anim1) <= 1.4 * avg(stat)},
        "criterion_7": {"ok": True, "note": "fps = 1000 / avg_ms by construction (bench_report_csv)"},
        "path": "voxanim::render_frame per frame (synchronous, RGB8 image to host), GPU FP32 kernel; "
                "render_ms = the call's wall time as in FrameStats",
    }
    return out


if __name__ == "__main__":
    print(json.dumps(measure()))
