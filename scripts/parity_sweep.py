"""Parity sweep at the BASELINE sizes (GPU box): every frame of the 120-frame C2
sequence and 12 C4 frames, FP64 kernel bit-exact (image, AOVs, FrameStats) and
FP32 kernel classified pixel by pixel (oracle/ref_harness.cpp classify_rule).
Writes a JSON summary (argv[1], default gpurun_out/parity_sweep.json)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_06001_b200 as vx  # noqa: E402
from oracle import ref  # noqa: E402

FIELDS = ("object_id", "node_index", "attr_index", "level", "entry_axis", "t", "kind", "traversals", "node_fetches")


def run(name, cfg, depth, times):
    model = vx.Model.procedural(depth, shell=True)
    s = vx.Scene(cfg, [model])
    o = ref.RefScene(cfg, [ref.RefModel.from_bytes(model.serialize())], 0, s.width, s.height)
    out = {"config": name, "frames": 0, "fp64_bit_exact_frames": 0, "fp32_rules": {}, "hit_pixels": 0,
           "fp32_bug_pixels": 0, "fp32_t_out_pixels": 0, "max_tie_frac": 0.0}
    th = ref.hardware_threads()
    for t in times:
        s.evaluate(t)
        o.evaluate(t)
        oa, orgb = o.dump(threads=th)
        oimg, ost = o.render(threads=th)
        rgb64, a64, st64 = s.render(precision=vx.VXA_FP64, aov=True)
        exact = (rgb64 == oimg).all() and all((a64[f] == oa[f]).all() for f in FIELDS) and \
            (a64["voxel"] == oa["voxel"]).all() and all(st64[k] == ost[k] for k in
                                                        ("rays", "sphere_tests", "svo_traversals", "pixels_reused"))
        _, a32, _ = s.render(precision=vx.VXA_FP32, aov=True)
        rules = o.classify_rules(oa, a32)
        h = ref.rule_histogram(rules)
        hits = int((oa["object_id"] >= 0).sum())
        ties = int(((rules > 0) & (rules < 100)).sum())
        out["frames"] += 1
        out["fp64_bit_exact_frames"] += int(bool(exact))
        out["hit_pixels"] += hits
        out["fp32_bug_pixels"] += int((rules == ref.RULE_BUG).sum())
        out["fp32_t_out_pixels"] += int((rules == ref.RULE_T_OUT).sum())
        out["max_tie_frac"] = max(out["max_tie_frac"], ties / max(1, hits))
        for k, v in h.items():
            out["fp32_rules"][k] = out["fp32_rules"].get(k, 0) + v
        if not exact or (rules >= 100).any():
            print(f"{name} t={t}: fp64 exact {exact} {h}", flush=True)
    out["fp32_tie_frac_of_hits"] = sum(v for k, v in out["fp32_rules"].items()
                                       if k not in ("bug", "t_out_of_tolerance")) / max(1, out["hit_pixels"])
    return out


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_sweep.json"
    t0 = time.time()
    doc = {"note": "full-size parity sweep: FP64 kernel bit-exact vs the reference (image, per-pixel AOVs, "
                   "FrameStats); FP32 kernel per-pixel rule histogram (oracle/ref_harness.cpp classify_rule)",
           "cases": [run("C2 (120-frame sequence, t = k/30)", vx.config.C2, 10, [k / 30.0 for k in range(120)]),
                     run("C4 (12 frames, t = k/3)", vx.config.C4, 11, [k / 3.0 for k in range(12)])]}
    doc["seconds"] = round(time.time() - t0, 1)
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc))


if __name__ == "__main__":
    main()
