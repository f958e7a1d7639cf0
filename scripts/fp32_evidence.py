"""FP32 parity evidence at the BASELINE sizes (run on the GPU box).

For full-size C2 (1920x1080, depth 10, animated) and C4 (3840x2160, 64 animated
depth-11 instances) frames at several animation times: the per-rule histogram
of the FP32 kernel's differences from the oracle (oracle/ref_harness.cpp
classify_rule), the t error distribution of matching hits, and the FP32
FrameStats / HitKind next to the reference's. Writes one JSON document
(argv[1], default gpurun_out/fp32_evidence.json).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_06001_b200 as vx  # noqa: E402
from oracle import ref  # noqa: E402

CASES = [("C2", vx.config.C2, 10, (0.0, 1.7, 3.3)), ("C4", vx.config.C4, 11, (0.4, 2.3, 3.6))]


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fp32_evidence.json"
    doc = {"note": "FP32 production kernel vs the reference oracle, full-size frames; rules: oracle/ref_harness.cpp "
                   "classify_rule", "cases": []}
    for name, cfg, depth, times in CASES:
        model = vx.Model.procedural(depth, shell=True)
        om = ref.RefModel.from_bytes(model.serialize())
        s = vx.Scene(cfg, [model])
        o = ref.RefScene(cfg, [om], 0, s.width, s.height)
        for t in times:
            t0 = time.time()
            s.evaluate(t)
            o.evaluate(t)
            o_aov, _ = o.dump(threads=ref.hardware_threads())
            o_img, o_st = o.render(threads=ref.hardware_threads())
            rgb, aov, st = s.render(precision=vx.VXA_FP32, aov=True)
            prod = s.render(precision=vx.VXA_FP32)[0]  # the production (no-AOV) instantiation
            rules = o.classify_rules(o_aov, aov)
            hit = o_aov["object_id"] >= 0
            match = rules == 0
            both = match & hit
            rel = np.abs(aov["t"][both] - o_aov["t"][both]) / np.maximum(1.0, np.abs(o_aov["t"][both]))
            diff = np.abs(rgb.astype(int) - o_img.astype(int)).max(axis=2)
            kind_bad = (aov["kind"] != o_aov["kind"]) & match
            case = {
                "config": name, "t": t, "width": s.width, "height": s.height,
                "hit_pixels": int(hit.sum()),
                "rules": ref.rule_histogram(rules),
                "tie_frac_of_hits": float(((rules > 0) & (rules < 100)).sum() / max(1, hit.sum())),
                "t_rel_err": {"max": float(rel.max()) if rel.size else 0.0,
                              "p999": float(np.quantile(rel, 0.999)) if rel.size else 0.0,
                              "mean": float(rel.mean()) if rel.size else 0.0},
                "rgb_max_lsb_on_matches": int(diff[match].max()) if match.any() else 0,
                "rgb_pixels_off_by_1_on_matches": int((diff[match] == 1).sum()),
                "stats": {"reference": {k: int(o_st[k]) for k in ("rays", "sphere_tests", "svo_traversals",
                                                                 "pixels_reused")},
                          "fp32": {k: int(st[k]) for k in ("rays", "sphere_tests", "svo_traversals",
                                                          "pixels_reused")}},
                "kind_mismatch_on_matching_pixels": int(kind_bad.sum()),
                "production_vs_aov_kernel_pixels_differ": int((prod != rgb).any(axis=2).sum()),
                "per_pixel_traversals_fp32_minus_ref": {
                    "more": int((aov["traversals"] > o_aov["traversals"]).sum()),
                    "fewer": int((aov["traversals"] < o_aov["traversals"]).sum())},
                "seconds": round(time.time() - t0, 1),
            }
            print(json.dumps(case), flush=True)
            doc["cases"].append(case)
    os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
    with open(out_path, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
