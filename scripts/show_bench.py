"""Print the key fields of gpurun_out/bench*.log lines (helper for A/B runs)."""
import glob
import json
import sys

for f in sys.argv[1:] or sorted(glob.glob("gpurun_out/bench*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            e2e = d.get("e2e") or {}
            print(f"{f:40s} {d['value']:9.1f} Mrays/s  {d['ms_per_step']:.4f} ms/step  kernel "
                  f"{d['roofline']['kernel_ms']:.4f} ms  e2e {e2e.get('value')}  launches {d.get('gpu_launches')}")
