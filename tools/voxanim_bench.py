"""`voxanim bench` on the GPU path: the reference CLI's bench modes and CSV report
(proj/src/cli.cpp:225-312, cmd_bench / bench_report_csv) for the benchmark
configurations, so its numbers line up with the reference's own tool.

Modes (cli.cpp:238-245): static = no animation, no optimisations; animated =
evaluate_animation(frame / fps) with culling, sorting and the hit buffer off;
animated-opt = animation with all three on. Per frame: render_frame, then
mark_clean (after one untimed warm-up render); the CSV repeats the counter totals on every row and ends with a
`mode,avg_ms,fps` summary line, numbers formatted like std::to_chars.

    python tools/voxanim_bench.py --config 2 --mode animated-opt --frames 60 --csv out.csv
"""
from __future__ import annotations

import argparse
import decimal
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CSV_HEADER = "mode,frame,ms,rays,sphere_tests,svo_traversals,pixels_reused"


def format_double(v: float) -> str:
    """std::to_chars(double) shortest form (cli.cpp:30-34): the shortest
    round-trip digits, printed as %f or %e whichever is shorter (%f on a tie)."""
    if v != v or v in (float("inf"), float("-inf")):
        return {True: "nan"}.get(v != v, "inf" if v > 0 else "-inf")
    if v == 0.0:
        return "-0" if str(v).startswith("-") else "0"
    sign, digits, exp = decimal.Decimal(repr(v)).normalize().as_tuple()
    ds = "".join(map(str, digits))
    n = len(ds)
    point = n + exp  # decimal point position relative to the digit string
    if point <= 0:
        fixed = "0." + "0" * (-point) + ds
    elif point >= n:
        fixed = str(abs(int(v)))  # %f form of an integral value: its exact digits
    else:
        fixed = ds[:point] + "." + ds[point:]
    e = point - 1
    sci = ds[0] + ("." + ds[1:] if n > 1 else "") + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"
    out = fixed if len(fixed) <= len(sci) else sci
    return ("-" if sign else "") + out


def bench_report_csv(mode: str, per_frame_ms, totals: dict) -> str:
    lines = [CSV_HEADER]
    for frame, ms in enumerate(per_frame_ms):
        lines.append(f"{mode},{frame},{format_double(ms)},{totals['rays']},{totals['sphere_tests']},"
                     f"{totals['svo_traversals']},{totals['pixels_reused']}")
    avg = sum(per_frame_ms) / len(per_frame_ms)
    lines.append(f"{mode},{format_double(avg)},{format_double(1000.0 / avg)}")
    return "\n".join(lines) + "\n"


def model_for(vx, config: int):
    if config == 1:
        words, gd = vx.grid_primitive("sphere", 8)
        return vx.Model.from_grid(words, gd)  # C1: the reference's dense sphere, built on the device
    if config in (2, 3):
        return vx.Model.procedural(10, shell=True)
    return vx.Model.procedural(11, shell=True)


def run_mode(vx, scene, mode: str, frames: int, fps: float, width: int, height: int):
    """cmd_bench's frame loop (cli.cpp:248-278) on one scene: returns (per-frame ms, counter totals)."""
    animate = mode != "static"
    opt = mode == "animated-opt"
    hbo = vx.HitBuffer(width, height) if opt else None
    # One untimed render first: the device context, the model's one-time
    # upload to HBM and the first launch of the kernel variant are not frame
    # costs (a throwaway hit buffer, no mark_clean: the scene's dirty state and
    # the timed HBO are untouched).
    scene.render(culling=opt, sorting=opt, hbo=vx.HitBuffer(width, height) if opt else None)
    per_frame, totals = [], {"rays": 0, "sphere_tests": 0, "svo_traversals": 0, "pixels_reused": 0}
    for frame in range(frames):
        if animate:
            scene.evaluate(frame / fps)
        _, _, st = scene.render(culling=opt, sorting=opt, hbo=hbo)
        scene.mark_clean()
        per_frame.append(st["render_ms"])
        for k in totals:
            totals[k] += int(st[k])
    return per_frame, totals


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--config", type=int, default=2, help="benchmark configuration (1-4, SURVEY.md §8(d))")
    ap.add_argument("--scene", default=None, help="a scene document (voxanim::load_scene_file) instead of --config")
    ap.add_argument("--mode", default="static", choices=["static", "animated", "animated-opt"])
    ap.add_argument("--frames", type=int, default=60)
    ap.add_argument("--width", type=int, default=640)
    ap.add_argument("--height", type=int, default=480)
    ap.add_argument("--fps", type=float, default=30.0)
    ap.add_argument("--csv", default=None, help="write the CSV report here (default: stdout)")
    args = ap.parse_args(argv)
    if args.frames < 1:
        raise SystemExit("frame count must be at least 1")
    if not args.fps > 0.0:
        raise SystemExit("fps must be positive")

    import paper_1911_06001_b200 as vx

    if args.scene:
        scene = vx.Scene.load(args.scene, args.width, args.height)
    else:
        scene = vx.Scene(args.config, [model_for(vx, args.config)], 0, args.width, args.height)
    per_frame, totals = run_mode(vx, scene, args.mode, args.frames, args.fps, args.width, args.height)
    text = bench_report_csv(args.mode, per_frame, totals)
    if args.csv:
        with open(args.csv, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
