#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (tracked).

    python scripts/summarize_profiles.py --tag r1 --full gpurun_out/x.ncu-rep [...]
                                         [--launches gpurun_out/launches.csv]
                                         [--traffic-kernel 'bk5_pencil<8']

Writes profiles/<tag>_ncu_<kernel>.json (key metrics + stall shares),
profiles/<tag>_launches.json (per-kernel launch counts / mean / share of a
BP5 iteration) and, for --traffic-kernel, profiles/bk5_traffic.json which
bench.py reports as roofline.traffic.
"""

import argparse
import collections
import csv
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]


def to_num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return v


def full_capture(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")], "source": os.path.basename(rep)}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = {"value": to_num(r[i]), "unit": units[i]}
        st = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): to_num(r[i])
              for i, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")}
        st = {k: v for k, v in st.items() if isinstance(v, float)}
        tot = sum(st.values()) or 1.0
        d["stall_share_pct"] = {k: round(100 * v / tot, 1)
                                for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
        res.append(d)
    return res


def scale(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return v * f


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = re.sub(r"\(.*", "", d["Kernel Name"]).strip()
        v = to_num(d["Metric Value"])
        u = d["Metric Unit"]
        v = v / 1000.0 if u == "ns" else (v * 1000.0 if u == "ms" else v)
        agg.setdefault(k, []).append(v)
    return {k: {"launches": len(v), "mean_us": round(sum(v) / len(v), 2),
                "min_us": round(min(v), 2), "total_us": round(sum(v), 1)} for k, v in agg.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--launches", default=None)
    ap.add_argument("--traffic-kernel", default=None)
    args = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    for rep in args.full:
        for d in full_capture(rep):
            short = re.sub(r"[^A-Za-z0-9_]+", "_", d["kernel"].split("(")[0].replace("void ", ""))
            short = short.strip("_")[:60]
            p = os.path.join(PROF, f"{args.tag}_ncu_{short}.json")
            json.dump(d, open(p, "w"), indent=1)
            print("wrote", p)
            # prefix match on the demangled name ("bk5_pencil<8" must not pick
            # up bk5_pencil_tma_pcg<8, 3>, the fused BP5 step)
            name = d["kernel"].split("(")[0].replace("void ", "").strip()
            if args.traffic_kernel and name.startswith(args.traffic_kernel):
                rd = d["dram__bytes_read.sum"]
                wr = d["dram__bytes_write.sum"]
                tr = scale(rd["value"], rd["unit"]) + scale(wr["value"], wr["unit"])
                json.dump({"kernel": d["kernel"].split("(")[0], "dram_bytes_per_launch": int(tr),
                           "dram_read": int(scale(rd["value"], rd["unit"])),
                           "dram_write": int(scale(wr["value"], wr["unit"])),
                           "source": f"profiles/{args.tag}_ncu_{short}.json (ncu --set full)"},
                          open(os.path.join(PROF, "bk5_traffic.json"), "w"), indent=1)
    if args.launches:
        L = launches(args.launches)
        p = os.path.join(PROF, f"{args.tag}_launches.json")
        json.dump(L, open(p, "w"), indent=1)
        print("wrote", p)


if __name__ == "__main__":
    main()
