"""Summarise one kernel of an `ncu --set full` report into JSON (the counters
DESIGN.md cites: time, DRAM / L2 / L1 traffic and hit rates, issue and pipe
utilisation, lane activity (divergence), occupancy, registers, spills).

    python scripts/ncu_summary.py profiles/r1_frame_kernel_c4.ncu-rep c4 profiles/ncu_frame_kernel.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "kernel_ms_under_ncu": ("gpu__time_duration.sum", 1e-0),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "l2_sectors": ("lts__t_sectors.sum", None),
    "l2_hit_rate_pct": ("lts__t_sector_hit_rate.pct", None),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", None),
    "l1_hit_rate_pct": ("l1tex__t_sector_hit_rate.pct", None),
    "global_load_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", None),
    "local_store_sectors": ("l1tex__m_l1tex2xbar_write_sectors_mem_lg_op_st.sum", None),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", None),
    "alu_pipe_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", None),
    "fma_pipe_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", None),
    "active_lanes_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", None),
    "warp_instructions": ("smsp__inst_executed.sum", None),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "registers": ("launch__registers_per_thread", None),
    "grid": ("launch__grid_size", None),
    "block": ("launch__block_size", None),
}
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
         "nsecond": 1e-6, "ns": 1e-6}


def summarise(rep: str) -> dict:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    out = {"kernel": v[h.index("Kernel Name")]}
    for key, (m, _) in METRICS.items():
        if m not in h:
            continue
        i = h.index(m)
        x = float(v[i].replace(",", ""))
        x *= SCALE.get(units[i], 1.0)
        out[key] = round(x, 6) if x < 1e6 else int(x)
    out["dram_bytes_per_launch"] = int(out.get("dram_read_bytes", 0) + out.get("dram_write_bytes", 0))
    if "l2_sectors" in out:
        out["l2_bytes"] = int(out["l2_sectors"] * 32)
    return out


if __name__ == "__main__":
    rep, key, dst = sys.argv[1], sys.argv[2], sys.argv[3]
    s = summarise(rep)
    s["source"] = f"ncu --set full --clock-control none ({rep})"
    try:
        with open(dst) as f:
            doc = json.load(f)
    except FileNotFoundError:
        doc = {}
    doc[key] = s
    with open(dst, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(s, indent=1))
