#!/usr/bin/env python
"""voxanim-b200 benchmark: animated-SVO ray casting, SURVEY.md §8(d) configuration C4.

A step is one animated frame of 64 rigid-body-animated instances of one
depth-11 shell-sphere SVO at 3840x2160 (8,294,400 primary rays): the host
update (evaluate_animation + instance table) and the GPU frame (ray
generation, bounding-sphere cull + front-to-back order, Revelles traversal,
nearest hit, shading, RGBA8 store). N GPUs split the frame into 64x64
super-tiles (round-robin) and store their tiles straight into rank 0's
framebuffer over NVLink (CUDA IPC peer mapping): strong scaling.

Prints ONE JSON line on rank 0. --impl reference runs the reference CPU
renderer (oracle/_ref, compiled from /root/reference) on the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (config id, shell?, depth, width, height, animated)
    "c4": (4, True, 11, 3840, 2160, True),
    "c2": (2, True, 10, 1920, 1080, True),
    "c3": (3, True, 10, 1920, 1080, False),
    "c1": (1, False, 8, 512, 512, False),
}
WORKLOAD_TEXT = {
    "c4": "C4: 64 animated instances of a depth-11 shell-sphere SVO, 3840x2160, culling+sorting, nearest hit",
    "c2": "C2: one depth-10 shell-sphere SVO animated (rotation+translation+anisotropic scale), 1920x1080",
    "c3": "C3: C2's model and camera, static identity transform",
    "c1": "C1: static depth-8 solid sphere, identity transform, 512x512",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-flush", action="store_true", help="do not flush L2 between timed steps")
    ap.add_argument("--headstart-us", type=int, default=500,
                    help="stream delay before each timed step (host enqueue latency stays out of device time)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the cpu_baseline sample")
    ap.add_argument("--no-extras", action="store_true", help="skip the C2/C3 animated-vs-static side measurements")
    ap.add_argument("--same-device", action="store_true",
                    help="testing aid: every rank uses GPU 0 (CUDA IPC between processes on one device, gloo "
                         "barriers) to exercise the multi-rank path on a one-GPU box; not a scaling measurement")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


# ---------------------------------------------------------------------------- clocks

class ClockSampler:
    """SM clocks + throttle reasons (NVML every 5 ms, nvidia-smi as the fallback), sampled in the
    background during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._first = threading.Event()  # set once a sample exists (NVML start-up can take ~1 s)
        self._t = None

    # NVML clocks-event reason bits (nvml.h: nvmlClocksEventReason*)
    NVML_BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4}

    def _poll_nvml(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                bits = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append([str(sm), str(mx)] +
                                    ["Active" if bits & self.NVML_BITS[n] else "Not Active" for n in self.NAMES])
                self._first.set()
                self._stop.wait(0.005)
        finally:
            pynvml.nvmlShutdown()

    def _poll(self):
        try:
            import pynvml  # noqa: F401  (nvidia_ml_py)
            return self._poll_nvml()
        except Exception:
            self.samples = []
        cmd = ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
               "--format=csv,noheader,nounits"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(cmd, capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
                    self._first.set()
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._poll, daemon=True)
        self._t.start()
        # the timed region starts only once the sampler is running, so even a short run is covered
        self._first.wait(timeout=20)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = set()
        for s in self.samples:
            for name, v in zip(self.NAMES, s[2:]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------- helpers

def crowd_bench(lib, ctx, vxl, prec, count: int = 4096, frames: int = 60) -> dict:
    """4096 animated instances of a depth-8 shell at
    3840x2160 (config CROWD). Device time per frame (CUDA events, L2 flushed)
    and the host time of the per-frame scene update (evaluate_animation of 4096
    tracks + the FP64 instance table + launch), measured around
    vxn_scene_submit, which returns once the frame is enqueued."""
    import paper_1911_06001_b200 as vx
    from paper_1911_06001_b200 import _abi
    sc = vx.Scene(vx.config.CROWD, [vx.Model.procedural(8, shell=True)], count)
    for k in range(5):
        vxl.vxn_scene_submit(sc._h, k / 30.0, prec, 0, 1, 0)
    lib.vxa_synchronize(ctx)
    lib.vxa_stats_reset(ctx)
    dev, host = [], []
    for k in range(frames):
        lib.vxa_flush_l2(ctx)
        lib.vxa_synchronize(ctx)
        lib.vxa_timer_begin(ctx)
        t0 = time.perf_counter()
        if vxl.vxn_scene_submit(sc._h, (5 + k) / 30.0, prec, 0, 1, 0) != 0:
            raise RuntimeError(vxl.vxn_last_error().decode())
        host.append((time.perf_counter() - t0) * 1e3)
        ms = C.c_double()
        lib.vxa_timer_end(ctx, C.byref(ms))
        dev.append(ms.value)
    st = _abi.vxa_stats()
    lib.vxa_stats_read(ctx, C.byref(st))
    # pipelined: the host update of frame k+1 overlaps frame k on the GPU (no
    # per-frame sync; double-buffered instance staging), wall clock per frame
    lib.vxa_synchronize(ctx)
    t0 = time.perf_counter()
    for k in range(frames):
        lib.vxa_flush_l2(ctx)
        if vxl.vxn_scene_submit(sc._h, (100 + k) / 30.0, prec, 0, 1, 0) != 0:
            raise RuntimeError(vxl.vxn_last_error().decode())
    lib.vxa_synchronize(ctx)
    pipelined = (time.perf_counter() - t0) * 1e3 / frames
    kern = st.gpu_ms / frames  # per-frame kernel events (pre-pass + frame kernel)
    msf = statistics.mean(dev)
    return {"instances": count, "kernel_ms_per_frame": round(kern, 4),
            "mrays_per_s_kernel": round(3840 * 2160 / kern / 1e3, 1),
            "step_ms_per_frame": round(msf, 4),
            "step_note": "events around vxn_scene_submit: host update (GPU idle) + H2D + kernels",
            "host_update_ms_per_frame": round(statistics.median(host), 4),
            "pipelined_ms_per_frame": round(pipelined, 4),
            "pipelined_note": "wall clock, frame k+1's host update overlapping frame k's kernels, L2 flushed",
            "kernel_launches_per_frame": round(st.kernel_launches / frames, 2),
            "traversals_per_ray": round(st.svo_traversals / (frames * 3840 * 2160), 4),
            "node_fetches_per_ray": round(st.node_fetches / (frames * 3840 * 2160), 4), "frames": frames}


def partition_shares(lib, ctx, vxl, scene, animated, args, W, H, frames: int = 8) -> dict:
    """C4 rendered as rank r of N (64x64 super-tiles dealt round-robin, the
    multi-GPU partition) on this one GPU: the device time (CUDA events, L2 flushed)
    of every rank's share, per N. max over ranks bounds an N-GPU frame's compute;
    t1 / (N * max) is the strong-scaling efficiency that partition allows before
    the composition and the frame flags."""
    from paper_1911_06001_b200 import _abi

    def share_ms(rank, world):
        for k in range(2):
            vxl.vxn_scene_submit(scene._h, frame_time(k, animated), _abi.VXA_FP32, rank, world, 0)
        lib.vxa_synchronize(ctx)
        tot = 0.0
        for k in range(frames):
            lib.vxa_flush_l2(ctx)
            lib.vxa_stream_delay(ctx, args.headstart_us)
            lib.vxa_timer_begin(ctx)
            if vxl.vxn_scene_submit(scene._h, frame_time(args.warmup + k, animated), _abi.VXA_FP32, rank, world, 0) != 0:
                raise RuntimeError(vxl.vxn_last_error().decode())
            ms = C.c_double()
            lib.vxa_timer_end(ctx, C.byref(ms))
            tot += ms.value
        return tot / frames

    t1 = share_ms(0, 1)
    out = {"frames_per_share": frames, "n1_ms": round(t1, 4)}
    for n in (2, 4, 8):
        per = [share_ms(r, n) for r in range(n)]
        out[f"n{n}"] = {"rank_ms": [round(x, 4) for x in per], "max_ms": round(max(per), 4),
                        "compute_efficiency": round(t1 / (n * max(per)), 3)}
    out["note"] = ("one GPU renders each rank's super-tiles in turn (vxn_scene_submit rank/world); the N-GPU "
                   "frame adds the NVLink composition and the device-side frame flags")
    return out


def model_build_bench(lib, ctx, reps: int = 5) -> dict:
    """build_from_grid on the device (vxa_build_model)
    for the reference's dense sphere grid at depth 10 (1024^3 bitset, 128 MiB,
    page-locked host memory; timed: H2D of the grid + every build kernel), next
    to the product's host builder at depth 10 and the reference's own
    build_from_grid at depth 8 (C1's model; at depth 10 it needs ~48 s / 15 GB)."""
    import paper_1911_06001_b200 as vx

    def check(rc, what):
        if rc != 0:
            raise RuntimeError(f"{what}: {lib.vxa_last_error().decode()}")

    out = {}
    for depth in (8, 10):
        words, gd = vx.grid_primitive("sphere", depth)
        check(lib.vxa_host_register(ctx, words.ctypes.data, words.nbytes), "host_register")
        times = []
        h, nn, na = C.c_uint32(), C.c_uint64(), C.c_uint64()
        for _ in range(reps + 1):
            t0 = time.perf_counter()
            check(lib.vxa_build_model(ctx, words.ctypes.data, gd, 0, 0, C.byref(h), C.byref(nn), C.byref(na)),
                  "build_model")
            times.append((time.perf_counter() - t0) * 1e3)
            lib.vxa_release_model(ctx, h.value)
        lib.vxa_host_unregister(ctx, words.ctypes.data)
        row = {"grid_bytes": int(words.nbytes), "nodes": nn.value, "attributes": na.value,
               "device_ms": round(statistics.median(times[1:]), 3)}
        t0 = time.perf_counter()
        vx.Model.from_grid(words, gd, device=False)
        row["host_builder_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
        if depth == 8:
            from oracle import ref  # CPU baseline of this row: the reference itself
            t0 = time.perf_counter()
            ref.RefModel.dense_sphere(8)  # gen_primitive + build_from_grid (gen is ~5% of it)
            row["reference_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
        out[f"sphere_depth{depth}"] = row
    out["path"] = ("vxa_build_model: grid H2D, Morton leaf masks, mask pyramid, per-level popcount, "
                   "exclusive scan, emission of 12-byte records + compact words + attributes, wide repack")
    return out


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def ncu_traffic(workload):
    """DRAM bytes per frame-kernel launch from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_frame_kernel.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    e = d.get(workload)
    return e.get("dram_bytes_per_launch") if e else None


def ncu_compute(workload):
    """Issue-side utilisation of the frame kernel from the same committed ncu
    summary: the kernel is issue-bound, which the HBM fraction alone hides."""
    p = os.path.join(ROOT, "profiles", "ncu_frame_kernel.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        e = json.load(f).get(workload)
    if not e or "issue_active_pct" not in e:
        return None
    return {"bound": "instruction issue", "issue_active_pct": e["issue_active_pct"],
            "alu_pipe_pct": e.get("alu_pipe_pct"), "active_lanes_per_inst": e.get("active_lanes_per_inst"),
            "source": "profiles/ncu_frame_kernel.json (ncu --set full)"}


def exchange_gpu_ids(rank: int, world: int, device: int) -> list:
    """UUIDs of every rank's GPU, exchanged through a TCP store beside the process group's
    rendezvous (before any backend is chosen)."""
    import datetime

    import torch
    import torch.distributed as dist

    store = dist.TCPStore(os.environ.get("MASTER_ADDR", "127.0.0.1"), int(os.environ.get("MASTER_PORT", "29500")) + 1,
                          world, rank == 0, timeout=datetime.timedelta(seconds=120))
    store.set(f"gpu{rank}", str(torch.cuda.get_device_properties(device).uuid))
    ids = [store.get(f"gpu{r}").decode() for r in range(world)]
    store.set(f"done{rank}", "1")
    if rank == 0:  # the server outlives every client's last read
        for r in range(world):
            store.get(f"done{r}")
    return ids


def exchange_handle(dist, rank, handle: bytes) -> bytes:
    """Broadcast rank 0's 64-byte CUDA IPC framebuffer handle to every rank."""
    obj = [handle if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def build_scene(vx, workload):
    cfg, shell, depth, W, H, animated = WORKLOADS[workload]
    model = vx.Model.procedural(depth, shell=shell)
    scene = vx.Scene(cfg, [model])
    return model, scene, W, H, animated


def frame_time(k, animated):
    return ((k / 30.0) % 4.0) if animated else 0.0


def cpu_baseline(model, workload, seconds, max_frames=5):
    """Reference render_frame (oracle/_ref, all host threads) on a bounded sample of the workload."""
    from oracle import ref

    cfg, shell, depth, W, H, animated = WORKLOADS[workload]
    rmodel = ref.RefModel.from_bytes(model.serialize())
    rscene = ref.RefScene(cfg, [rmodel], 0, W, H)
    threads = ref.hardware_threads()
    total_ms, frames = 0.0, 0
    t0 = time.perf_counter()
    while frames < max_frames and (frames == 0 or time.perf_counter() - t0 < seconds):
        rscene.evaluate(frame_time(frames, animated))
        _, st = rscene.render(True, True, threads)
        total_ms += st["render_ms"]
        frames += 1
    value = W * H * frames / (total_ms / 1e3) / 1e6
    return {"value": round(value, 4), "unit": "Mrays/s", "cores": threads, "kind": "reference",
            "sample": f"{frames} full {W}x{H} frames of {workload.upper()} (t=k/30), reference render_frame "
                      f"(culling+sorting, no HBO), FrameStats::render_ms",
            "ms_per_frame": round(total_ms / frames, 3)}


def oracle_bytes(model, workload, ks):
    """Algorithmic bytes per ray counted by the ORACLE: the
    reference's own per-pixel internal-node visits (traverse_debug, replayed in
    shade_pixel's candidate order and skip rule by oracle/ref_harness.cpp's dump)
    x 8 B + 4 B per attribute fetch (hit) + 4 B framebuffer store, over full
    frames at the animation times of timed steps ks."""
    import numpy as np
    from oracle import ref

    cfg, shell, depth, W, H, animated = WORKLOADS[workload]
    rscene = ref.RefScene(cfg, [ref.RefModel.from_bytes(model.serialize())], 0, W, H)
    fetches = hits = trav = n = 0
    for k in ks:
        rscene.evaluate(frame_time(k, animated))
        aov, _ = rscene.dump(threads=ref.hardware_threads())
        fetches += int(aov["node_fetches"].astype(np.int64).sum())
        hits += int((aov["object_id"] >= 0).sum())
        trav += int(aov["traversals"].astype(np.int64).sum())
        n += aov.size
    return {"bytes_per_ray": (8.0 * fetches + 4.0 * hits + 4.0 * n) / n, "node_fetches_per_ray": fetches / n,
            "leaf_hits_per_ray": hits / n, "traversals_per_ray": trav / n,
            "sample": f"{len(ks)} full {W}x{H} frames at t = " + ", ".join(f"{frame_time(k, animated):.4f}" for k in ks)
                      + " s of the timed steps, reference traverse_debug visits (oracle/_ref dump)"}


# ---------------------------------------------------------------------------- reference arm

def reference_model(ref, workload):
    """The workload's model for the reference arm, loaded by the reference's own
    load_svo. The reference cannot build the depth-11 shell itself (its
    build_from_grid needs a 2048^3 grid and a pointer tree of tens of GB), so a
    CHILD process runs this repo's procedural builder -- pinned byte-identical to
    the reference build_from_grid of the same grid (tests/test_builder.py) -- and
    writes the .svo; this process only ever loads oracle/_ref."""
    import tempfile

    cfg, shell, depth, W, H, animated = WORKLOADS[workload]
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, f"model_d{depth}.svo")
        code = (f"import sys; sys.path.insert(0, {ROOT!r}); import paper_1911_06001_b200 as vx; "
                f"vx.Model.procedural({depth}, shell={shell}).save({path!r})")
        subprocess.run([sys.executable, "-c", code], check=True)
        return ref.RefModel.load(path)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import ref

    cfg, shell, depth, W, H, animated = WORKLOADS[args.workload]
    rmodel = reference_model(ref, args.workload)
    rscene = ref.RefScene(cfg, [rmodel], 0, W, H)
    threads = ref.hardware_threads()
    # First warm-up step: one full reference frame; it sizes the sample so the
    # whole run stays within a few minutes.
    rscene.evaluate(frame_time(0, animated))
    _, st = rscene.render(True, True, threads)
    full_ms = st["render_ms"]
    per_step_ms = 150e3 / max(1, args.steps + args.warmup)
    band = H if full_ms <= per_step_ms else max(8, min(H, int(H * per_step_ms / full_ms) // 8 * 8))

    def step(k):
        rscene.evaluate(frame_time(k, animated))
        if band == H:
            return rscene.render(True, True, threads)[1]["render_ms"]
        a = (k * band) % (H - band + 1)
        return rscene.render_rows(a, a + band, threads, rgb=False)[1]

    for k in range(1, args.warmup):
        step(k)
    total_ms = sum(step(args.warmup + k) for k in range(args.steps))
    ms = total_ms / args.steps
    value = W * band / ms / 1e3
    frame_ms = ms * H / band
    sample = (f"{args.steps} full {W}x{H} frames" if band == H else
              f"{args.steps} bands of {band} rows x {W} px (rotating, t=k/30) of the {W}x{H} frame")
    line = {
        "impl": "reference", "metric": "Mrays/s", "value": round(value, 4), "unit": "Mrays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "fps": round(1000.0 / frame_ms, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_TEXT[args.workload], "width": W, "height": H, "svo_depth": depth,
                   "instances": 64 if cfg == 4 else 1, "culling": True, "sorting": True, "hbo": False,
                   "l2": "n/a: CPU reference (the 108 MB model and 33 MB frame exceed the host caches)"},
        "cpu_baseline": {"value": round(value, 4), "unit": "Mrays/s", "cores": threads, "kind": "reference",
                         "sample": sample + f", reference render_frame/trace_ray on {threads} host threads"},
        "e2e": {"value": round(value, 4), "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- our arm

def run_ours(args):
    rank, world, local = dist_env()
    device = 0 if args.same_device else local
    if world > 1 and not args.same_device:
        import torch

        # a launcher that gives each process one visible GPU: LOCAL_RANK is not an ordinal there
        if torch.cuda.device_count() <= local:
            device = local = 0
        # more ranks than physical GPUs (e.g. --gpus 2 on a one-GPU box): NCCL cannot put two
        # ranks on one device, so run the shared-device path (gloo barriers, CUDA IPC) -- a
        # correctness run of the multi-rank path, labelled as such, not a scaling measurement
        try:
            ids = exchange_gpu_ids(rank, world, device)
        except Exception as e:  # no side channel: assume one GPU per rank, as before
            print(f"bench: GPU id exchange failed ({e}); assuming one GPU per rank", file=sys.stderr)
            ids = [str(r) for r in range(world)]
        if len(set(ids)) < world:
            args.same_device = True
            device = local = 0
            if rank == 0:
                print(f"bench: {world} ranks share fewer than {world} GPUs: shared-device mode", file=sys.stderr)
    os.environ["VOXANIM_DEVICE"] = str(device)
    import paper_1911_06001_b200 as vx
    from paper_1911_06001_b200 import _abi

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        if args.same_device:
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    lib = vx.vxa()
    model, scene, W, H, animated = build_scene(vx, args.workload)
    ctx = vx.context()
    f, inst, n = scene.export()
    prec = _abi.VXA_FP64 if args.precision == "fp64" else _abi.VXA_FP32

    def check(rc, what):
        if rc != 0:
            raise RuntimeError(f"{what}: {lib.vxa_last_error().decode()}")

    # multi-GPU: map rank 0's framebuffer into every rank (NVLink peer stores)
    composition = ("single device" if world == 1 else
                   "CUDA IPC stores into rank 0's framebuffer (ranks share one device)" if args.same_device else
                   "NVLink peer stores into rank 0's framebuffer (CUDA IPC)")
    if world > 1:
        handle = (C.c_char * 64)()
        if rank == 0:
            check(lib.vxa_fb_export(ctx, W, H, handle), "fb_export")
        got = exchange_handle(dist, rank, bytes(handle))
        ok = 1
        if rank != 0:
            h2 = (C.c_char * 64).from_buffer_copy(got)
            if lib.vxa_fb_import(ctx, W, H, h2) != 0:
                print(f"rank {rank}: vxa_fb_import failed ({lib.vxa_last_error().decode()}); "
                      "rendering into the local framebuffer", file=sys.stderr)
                ok = 0
        import torch
        t = torch.tensor([ok], dtype=torch.int32, device="cpu" if args.same_device else f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if int(t.item()) == 0 or os.environ.get("VOXANIM_COMPOSE") == "gather":
            # no CUDA IPC on every rank (or forced): compose by a collective gather instead
            if rank != 0:
                lib.vxa_fb_import(ctx, W, H, None)  # detach any peer mapping
            composition = ("collective gather: each rank packs its super-tiles (vxa_tiles_pack), "
                           "torch.distributed gather to rank 0, rank 0 unpacks them into its framebuffer")

    gather_buf = None
    if composition.startswith("collective"):
        import torch

        n_max = C.c_uint32()
        check(lib.vxa_tiles_count(W, H, 0, world, C.byref(n_max)), "tiles_count")  # rank 0 has the most
        dev = "cuda:0" if args.same_device else f"cuda:{local}"
        gather_buf = torch.zeros(n_max.value * 64 * 64, dtype=torch.int32, device=dev)
        gather_host = args.same_device  # gloo: the collective runs on host tensors

    # Frame completion without a host barrier (peer-store composition): rank 0
    # exports a flag block; every frame is opened by rank 0's go flag and closed
    # when every rank's done flag has landed in rank 0's HBM (vxa_frame_open /
    # vxa_frame_close). Ranks on distinct GPUs wait on the device (1-thread flag
    # kernels, system-scope acquire/release over NVLink); ranks sharing a GPU
    # must not run kernels that wait on one another, so there the same protocol
    # polls the flags from the host.
    sync = None
    if world > 1 and gather_buf is None:
        h = (C.c_char * 64)()
        if rank == 0:
            check(lib.vxa_sync_export(ctx, world, h), "sync_export")
        got = exchange_handle(dist, rank, bytes(h))
        if rank != 0:
            check(lib.vxa_sync_import(ctx, rank, world, (C.c_char * 64).from_buffer_copy(got)), "sync_import")
        sync = _abi.VXA_SYNC_HOST if args.same_device else _abi.VXA_SYNC_DEVICE
        check(lib.vxa_sync_configure(ctx, sync, 20000), "sync_configure")

    def gather_compose():
        """The frame's super-tiles of every rank into rank 0's framebuffer (gather mode)."""
        import torch

        gather_buf.zero_()
        torch.cuda.synchronize()
        check(lib.vxa_tiles_pack(ctx, W, H, rank, world, C.c_void_p(gather_buf.data_ptr())), "tiles_pack")
        check(lib.vxa_synchronize(ctx), "sync")
        send = gather_buf.cpu() if gather_host else gather_buf
        if rank == 0:
            parts = [torch.empty_like(send) for _ in range(world)]
            dist.gather(send, gather_list=parts, dst=0)
            for r in range(1, world):
                src = parts[r].to(gather_buf.device) if gather_host else parts[r]
                torch.cuda.synchronize()
                check(lib.vxa_tiles_unpack(ctx, W, H, r, world, C.c_void_p(src.data_ptr())), "tiles_unpack")
            check(lib.vxa_synchronize(ctx), "sync")
        else:
            dist.gather(send, dst=0)

    vxl = vx.voxanim()

    def submit(k):
        # host update (evaluate_animation) + instance table + frame submission, in C++
        if vxl.vxn_scene_submit(scene._h, frame_time(k, animated), prec, rank, world, 0) != 0:
            raise RuntimeError(vxl.vxn_last_error().decode())

    def barrier():
        if dist is not None:
            dist.barrier()

    def frame(k, timed=False):
        """One frame of this rank. N > 1 with flags: rank 0 opens it (go) and closes
        it when every rank's tiles have landed; rank r waits for go, renders, and
        signals done. The events bracket rank 0's whole frame (go .. last done)
        and rank r's own part. Gather mode: host-synchronised collective."""
        if sync is not None:
            if rank == 0:
                if timed:
                    check(lib.vxa_timer_begin(ctx), "timer")
                check(lib.vxa_frame_open(ctx), "frame_open")
            else:
                check(lib.vxa_frame_open(ctx), "frame_open")
                if timed:
                    check(lib.vxa_timer_begin(ctx), "timer")
            submit(k)
            check(lib.vxa_frame_close(ctx), "frame_close")
            return
        if timed:
            check(lib.vxa_timer_begin(ctx), "timer")
        submit(k)
        if gather_buf is not None:
            check(lib.vxa_synchronize(ctx), "sync")
            gather_compose()
            barrier()  # gather mode: the frame is complete when the collective is

    for k in range(args.warmup):
        frame(k)
    check(lib.vxa_synchronize(ctx), "sync")
    barrier()

    step_ms = []
    lib.vxa_stats_reset(ctx)
    with ClockSampler(local) as clocks:
        for k in range(args.steps):
            if not args.no_flush:
                check(lib.vxa_flush_l2(ctx), "flush")
            # the stream idles ~0.5 ms before the timed region opens, so the host has enqueued the
            # step's upload and kernels by then: the device time is the step's, not the host's
            # submission latency (which the e2e number carries). N > 1: rank 0's delay; the
            # other ranks' frames start at its go flag.
            if args.headstart_us > 0 and rank == 0:
                check(lib.vxa_stream_delay(ctx, args.headstart_us), "delay")
            frame(args.warmup + k, timed=True)
            ms = C.c_double()
            check(lib.vxa_timer_end(ctx, C.byref(ms)), "timer")
            step_ms.append(ms.value)
    st = _abi.vxa_stats()
    check(lib.vxa_stats_read(ctx, C.byref(st)), "stats")
    total_ms = sum(step_ms)

    def max_over_ranks(x):
        if dist is None:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cpu" if args.same_device else f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    total_ms = max_over_ranks(total_ms)

    ms_per_step = total_ms / args.steps
    rays = W * H
    value = rays * args.steps / (total_ms / 1e3) / 1e6

    # roofline of the frame kernel: algorithmic bytes / kernel time
    frames = max(1, st.frames)
    kernel_ms = st.gpu_ms / frames  # per frame: the culling pre-pass (if any) + the frame kernel
    pixels_mine = st.rays / frames
    alg_bytes = (8.0 * st.node_fetches + 4.0 * st.leaf_hits) / frames + 4.0 * pixels_mine
    peak, peak_src = measured_peaks()
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    traffic = ncu_traffic(args.workload)

    # N > 1: the frame composed in rank 0's framebuffer by peer stores must equal
    # the single-device frame (same pixels, same arithmetic)
    multi_ok = None
    if world > 1:
        import numpy as np

        barrier()
        k_chk = args.warmup + args.steps + 1
        frame(k_chk)
        check(lib.vxa_synchronize(ctx), "sync")
        barrier()
        if rank == 0:
            composed = np.empty((H, W, 3), np.uint8)
            check(lib.vxa_read_framebuffer(ctx, composed.ctypes.data, W, H), "read_framebuffer")
            if vxl.vxn_scene_submit(scene._h, frame_time(k_chk, animated), prec, 0, 1, 0) != 0:
                raise RuntimeError(vxl.vxn_last_error().decode())
            alone = np.empty((H, W, 3), np.uint8)
            check(lib.vxa_read_framebuffer(ctx, alone.ctypes.data, W, H), "read_framebuffer")
            multi_ok = bool((composed == alone).all())
        barrier()

    # end to end through the public API (voxanim::render_frame with host buffers)
    e2e = None
    if not args.no_e2e and world > 1:
        # every rank: host update + its super-tiles (peer stores into rank 0); rank 0
        # packs the composed frame once every rank's done flag is in and reads the RGB8
        # image into page-locked host memory on its copy stream while the next frame
        # renders (vxa_framebuffer_readback); no host barrier between frames
        import numpy as np

        bufs = [np.empty((H, W, 3), np.uint8) for _ in range(2)]
        if rank == 0:
            for b in bufs:
                check(lib.vxa_host_register(ctx, b.ctypes.data, b.nbytes), "host_register")
        lib.vxa_stats_reset(ctx)
        barrier()
        tickets = []
        ticket = C.c_uint64()
        t0 = time.perf_counter()
        for k in range(args.e2e_steps):
            frame(k)
            if rank == 0:
                check(lib.vxa_framebuffer_readback(ctx, W, H, bufs[k % 2].ctypes.data, C.byref(ticket)), "readback")
                tickets.append(ticket.value)
                if len(tickets) >= 2:
                    check(lib.vxa_wait_readback(ctx, tickets[-2]), "wait_readback")
        if rank == 0:
            check(lib.vxa_wait_readback(ctx, tickets[-1]), "wait_readback")
        check(lib.vxa_synchronize(ctx), "sync")
        el = max_over_ranks(time.perf_counter() - t0)
        st2 = _abi.vxa_stats()
        lib.vxa_stats_read(ctx, C.byref(st2))
        if rank == 0:
            for b in bufs:
                lib.vxa_host_unregister(ctx, b.ctypes.data)
        e2e = {"value": round(rays * args.e2e_steps / el / 1e6, 3), "unit": "Mrays/s",
               "h2d_bytes_per_step": int(st2.h2d_bytes // args.e2e_steps) * world,
               "d2h_bytes_per_step": W * H * 3, "ms_per_step": round(el * 1e3 / args.e2e_steps, 3),
               "path": "every rank: evaluate_animation + vxa_submit of its super-tiles (NVLink peer stores into "
                       "rank 0) between vxa_frame_open/close; rank 0: RGB8 pack of the composed frame + D2H "
                       "into a page-locked host image on its copy stream (overlapping the next frame)"
                       if sync is not None else
                       "every rank: evaluate_animation + vxa_submit; collective tile gather to rank 0; "
                       "rank 0: RGB8 pack + D2H"}
    sync_timeout = None
    if sync is not None:
        to = C.c_int32()
        check(lib.vxa_sync_status(ctx, C.byref(to)), "sync_status")
        sync_timeout = bool(max_over_ranks(float(to.value)))
        if sync_timeout:
            print(f"rank {rank}: a frame flag wait timed out", file=sys.stderr)
    if not args.no_e2e and world == 1:
        import numpy as np

        # page-locked caller images (vxa_host_register): per-frame D2H runs as DMA
        bufs = [np.empty((H, W, 3), np.uint8) for _ in range(2)]
        for b in bufs:
            check(lib.vxa_host_register(ctx, b.ctypes.data, b.nbytes), "host_register")
        # (1) synchronous: evaluate_animation + voxanim::gpu::render_frame_into per step
        for k in range(3):
            scene.evaluate(frame_time(k, animated))
            scene.render(precision=prec, rgb=bufs[0])
        t0 = time.perf_counter()
        for k in range(args.e2e_steps):
            scene.evaluate(frame_time(k, animated))
            scene.render(precision=prec, rgb=bufs[0])
        el_sync = time.perf_counter() - t0
        st2 = _abi.vxa_stats()
        lib.vxa_stats_read(ctx, C.byref(st2))
        h2d_step, d2h_step = int(st2.h2d_bytes), int(st2.d2h_bytes)
        # (2) streaming: frame k's RGB8 readback overlaps frame k+1's kernel
        #     (vxa_submit_readback); every step still uploads its instance table
        #     and lands its image in host memory inside the timed region
        tickets = []
        ticket = C.c_uint64()

        def stream(k):
            if vxl.vxn_scene_stream(scene._h, frame_time(k, animated), prec, bufs[k % 2].ctypes.data,
                                    C.byref(ticket)) != 0:
                raise RuntimeError(vxl.vxn_last_error().decode())
            tickets.append(ticket.value)
            if len(tickets) >= 2:
                check(lib.vxa_wait_readback(ctx, tickets[-2]), "wait_readback")

        for k in range(3):
            stream(k)
        check(lib.vxa_wait_readback(ctx, tickets[-1]), "wait_readback")
        tickets.clear()
        t0 = time.perf_counter()
        for k in range(args.e2e_steps):
            stream(k)
        check(lib.vxa_wait_readback(ctx, tickets[-1]), "wait_readback")
        el = time.perf_counter() - t0
        for b in bufs:
            lib.vxa_host_unregister(ctx, b.ctypes.data)
        # (3) the drop-in voxanim::render_frame: the Image returned by value (a fresh,
        #     zero-filled pageable vector) per call, evaluate_animation outside the calls
        ms_di = C.c_double()
        if vxl.vxn_scene_render_image(scene._h, frame_time(0, animated), 3, C.byref(ms_di), None) != 0:
            raise RuntimeError(vxl.vxn_last_error().decode())
        if vxl.vxn_scene_render_image(scene._h, frame_time(3, animated), args.e2e_steps, C.byref(ms_di), None) != 0:
            raise RuntimeError(vxl.vxn_last_error().decode())
        e2e = {"value": round(rays * args.e2e_steps / el / 1e6, 3), "unit": "Mrays/s",
               "h2d_bytes_per_step": h2d_step, "d2h_bytes_per_step": d2h_step,
               "ms_per_step": round(el * 1e3 / args.e2e_steps, 3),
               "path": "evaluate_animation + vxa_submit_readback per step: instance table H2D from pinned "
                       "staging, culling pre-pass + frame kernel (which also writes the RGB8 image), D2H "
                       "into a page-locked host image on a copy stream (overlapping the next frame's "
                       "kernel); wall clock over all steps",
               "sync": {"value": round(rays * args.e2e_steps / el_sync / 1e6, 3),
                        "ms_per_step": round(el_sync * 1e3 / args.e2e_steps, 3),
                        "path": "voxanim::gpu::render_frame_into into a page-locked image, one synchronous "
                                "call per step"},
               "drop_in": {"value": round(rays / ms_di.value / 1e3, 3), "ms_per_call": round(ms_di.value, 3),
                           "path": "voxanim::render_frame returning its Image by value (the reference's "
                                   "call), wall time per call"}}

    # side measurements: animated vs static at 1080p (configs C2 / C3)
    extras = None
    if rank == 0 and world == 1 and not args.no_extras:
        extras = {}
        m10 = vx.Model.procedural(10, shell=True)
        # "opt" = culling + sorting + the device-resident hit buffer (paper Fig. 6 "w/opt")
        runs = (("c2_animated_1080p", 2, True, False), ("c3_static_1080p", 3, False, False),
                ("c2_animated_opt_1080p", 2, True, True), ("c3_static_opt_1080p", 3, False, True),
                ("c4_1080p", 4, True, False))
        for name, cfg, anim, opt in runs:
            # C4 at 1080p: the 4K workload's 64 animated depth-11 instances, quarter the rays
            sc = vx.Scene(cfg, [model], 0, 1920, 1080) if cfg == 4 else vx.Scene(cfg, [m10])
            hbo = C.c_uint32(0)
            if opt:
                check(lib.vxa_hbo_create(ctx, 1920, 1080, C.byref(hbo)), "hbo_create")
            # BASELINE config 2: the whole 120-frame sequence at 30 fps (t = k/30, k = 0..119)
            steps_x = 120
            for k in range(steps_x - 5, steps_x):
                vxl.vxn_scene_submit(sc._h, frame_time(k, anim), prec, 0, 1, hbo.value)
            lib.vxa_synchronize(ctx)
            lib.vxa_stats_reset(ctx)
            tot = 0.0
            for k in range(steps_x):
                lib.vxa_flush_l2(ctx)
                lib.vxa_timer_begin(ctx)
                if vxl.vxn_scene_submit(sc._h, frame_time(k, anim) if anim else -1.0, prec, 0, 1, hbo.value) != 0:
                    raise RuntimeError(vxl.vxn_last_error().decode())
                msx = C.c_double()
                lib.vxa_timer_end(ctx, C.byref(msx))
                tot += msx.value
            stx = _abi.vxa_stats()
            lib.vxa_stats_read(ctx, C.byref(stx))
            if opt:
                lib.vxa_hbo_release(ctx, hbo.value)
            msf = tot / steps_x
            extras[name] = {"ms_per_frame": round(msf, 4), "fps": round(1000 / msf, 1),
                            "mrays_per_s": round(1920 * 1080 / msf / 1e3, 1), "frames": steps_x,
                            "sequence": "t = k/30 s, k = 0..119" if anim else "static",
                            "pixels_reused_per_frame": int(stx.pixels_reused // steps_x),
                            "traversals_per_frame": int(stx.svo_traversals // steps_x)}
        # the FP64 parity kernel (bit-exact vs the reference) on the headline workload
        if args.precision == "fp32" and args.workload == "c4":
            for k in range(3):
                vxl.vxn_scene_submit(scene._h, frame_time(k, animated), _abi.VXA_FP64, 0, 1, 0)
            lib.vxa_synchronize(ctx)
            lib.vxa_stats_reset(ctx)
            tot, nf = 0.0, 20
            for k in range(nf):
                lib.vxa_flush_l2(ctx)
                lib.vxa_stream_delay(ctx, args.headstart_us)
                lib.vxa_timer_begin(ctx)
                if vxl.vxn_scene_submit(scene._h, frame_time(args.warmup + k, animated), _abi.VXA_FP64, 0, 1, 0) != 0:
                    raise RuntimeError(vxl.vxn_last_error().decode())
                msx = C.c_double()
                lib.vxa_timer_end(ctx, C.byref(msx))
                tot += msx.value
            msf = tot / nf
            extras["c4_fp64"] = {"ms_per_frame": round(msf, 4), "fps": round(1000 / msf, 1),
                                 "mrays_per_s": round(W * H / msf / 1e3, 1), "frames": nf, "dtype": "f64",
                                 "note": "FP64 parity kernel (reference operation order, bit-exact image, AOVs "
                                         "and FrameStats), same workload, timing and L2 flush as value"}
        # the screen partition of the multi-GPU path, one rank's share at a time on this
        # GPU: per-rank device time of the C4 frame for N = 2, 4, 8 (the compute side of
        # strong scaling; composition over NVLink and the frame flags not included)
        if args.precision == "fp32" and args.workload == "c4":
            extras["partition_shares"] = partition_shares(lib, ctx, vxl, scene, animated, args, W, H)
        extras["animated_vs_static"] = round(extras["c2_animated_1080p"]["ms_per_frame"] /
                                             extras["c3_static_1080p"]["ms_per_frame"], 4)
        extras["model_build"] = model_build_bench(lib, ctx)
        extras["crowd_4096_4k"] = crowd_bench(lib, ctx, vxl, prec)

    orc = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            orc = oracle_bytes(model, args.workload,
                               [args.warmup + k * args.steps // 3 for k in range(3)] if animated else [0])
        except Exception as e:  # reported beside the kernel-counted bytes, not required
            print(f"bench: oracle byte count unavailable: {e}", file=sys.stderr)
    base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            base = cpu_baseline(model, args.workload, args.cpu_seconds)
        except Exception as e:  # the baseline is reported, not required
            base = {"value": None, "unit": "Mrays/s", "cores": None, "kind": "reference",
                    "sample": f"unavailable: {e}"}

    # the roofline's algorithmic bytes: oracle-counted per ray (the reference's
    # visits) x the rays of one launch; the kernel's own (pruned) counts beside it
    alg_bytes_o = orc["bytes_per_ray"] * pixels_mine if orc else alg_bytes
    achieved_o = alg_bytes_o / (kernel_ms / 1e3) / 1e9
    launches = int(st.kernel_launches)
    if dist is not None:  # every rank's kernels in the timed region
        import torch

        t = torch.tensor([launches], dtype=torch.int64, device="cpu" if args.same_device else f"cuda:{local}")
        dist.all_reduce(t)
        launches = int(t.item())
    timed_region = (f"CUDA events on the context stream around each step: culling pre-pass + frame kernel "
                    f"(the instance-table H2D is issued on the upload stream during the {args.headstart_us} us "
                    f"stream delay that precedes the region, so host enqueue latency and the upload stay out; "
                    f"e2e carries them)")
    if world > 1:
        timed_region += ("; N > 1: rank 0's events open before its go flag and close after every rank's done "
                         "flag, so they enclose every rank's frame and the flag exchange; value uses the max "
                         "over ranks")
    if rank == 0:
        cfg, shell, depth, _, _, _ = WORKLOADS[args.workload]
        line = {
            "metric": "Mrays/s", "value": round(value, 3), "unit": "Mrays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "fps": round(1000.0 / ms_per_step, 2), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT[args.workload], "width": W, "height": H, "svo_depth": depth,
                       "instances": 64 if cfg == 4 else 1, "culling": True, "sorting": True, "hbo": False,
                       "l2": "flushed between timed steps (256 MB write)" if not args.no_flush else "warm"},
            # how this arm ran the workload (kept out of `config`, which names the workload itself and
            # matches the reference arm's)
            "run": {"partition": (f"64x64 super-tiles round-robin over {world} ranks sharing one GPU "
                                  f"(multi-rank correctness run, not a scaling measurement)"
                                  if world > 1 and args.same_device else
                                  f"64x64 super-tiles round-robin over {world} GPU(s)"),
                    "composition": composition,
                    "timed_region": timed_region,
                    "frame_sync": (None if world == 1 else
                                   "device flags (vxa_frame_open/close: go/done flags in rank 0's HBM, 1-thread "
                                   "release/acquire kernels over NVLink, no host barrier)"
                                   if sync == _abi.VXA_SYNC_DEVICE else
                                   "host-polled flags (vxa_frame_open/close; ranks share one GPU)"
                                   if sync == _abi.VXA_SYNC_HOST else
                                   "host synchronisation + collective gather + barrier per frame")},
            "roofline": {"bound": "hbm", "achieved": round(achieved_o, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved_o / peak, 5), "traffic": traffic,
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": round(alg_bytes_o),
                         "algorithmic_bytes_source": ("oracle-counted (SURVEY.md §8(d)): " + orc["sample"]
                                                      if orc else "kernel-counted (no oracle sample at N > 1)"),
                         "algorithmic_bytes_oracle": round(alg_bytes_o) if orc else None,
                         "oracle_per_ray": ({k: round(v, 4) for k, v in orc.items() if k != "sample"}
                                            if orc else None),
                         "algorithmic_bytes_kernel_counted": round(alg_bytes),
                         "achieved_kernel_counted": round(achieved, 2),
                         "kernel_ms": round(kernel_ms, 4),
                         "per_ray": {"node_fetches": round(st.node_fetches / frames / pixels_mine, 4),
                                     "leaf_hits": round(st.leaf_hits / frames / pixels_mine, 4),
                                     "traversals": round(st.svo_traversals / frames / pixels_mine, 4),
                                     "bytes": round(alg_bytes / pixels_mine, 3)},
                         "compute": ncu_compute(args.workload)},
            "cpu_baseline": base,
            "e2e": e2e,
            "extras": extras,
            "gpu_launches": launches,
            "multi_gpu_frame_identical": multi_ok,
            "frame_sync_timed_out": sync_timeout,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 1 if sync_timeout else 0


def self_launch(args) -> int:
    """--gpus N > 1 without a launcher: start N ranks under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1) and return its exit code."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    rank, world, _ = dist_env()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if world != args.gpus:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
