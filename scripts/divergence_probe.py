"""Per-pixel work of the FP32 frame kernel at C4 (run on the GPU box).

Renders C4 frames through the AOV instantiation and saves each pixel's
traversal and node-fetch counts (uint16) plus its HitKind, so the SIMT
efficiency of the 8x4 warp tiles -- sum of the lanes' work over 32 x the
slowest lane's -- and of other tile shapes / refill schemes can be computed
off the box. Writes gpurun_out/divergence_c4.npz.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_06001_b200 as vx  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/divergence_c4.npz"
    model = vx.Model.procedural(11, shell=True)
    s = vx.Scene(vx.config.C4, [model])
    res = {}
    for k in (0, 37):
        s.evaluate((k / 30.0) % 4.0)
        _, aov, st = s.render(precision=vx.VXA_FP32, aov=True, rgb=False)
        res[f"fetch{k}"] = np.minimum(aov["node_fetches"], 65535).astype(np.uint16)
        res[f"trav{k}"] = np.minimum(aov["traversals"], 65535).astype(np.uint16)
        res[f"kind{k}"] = aov["kind"].astype(np.uint8)
        print(k, st, flush=True)
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    np.savez_compressed(out, **res)


if __name__ == "__main__":
    main()
