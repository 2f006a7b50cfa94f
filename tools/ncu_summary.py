#!/usr/bin/env python
"""Summarise ncu output into committed profile files (runs here, no GPU).

    python tools/ncu_summary.py --rep gpurun_out/prof_full.ncu-rep \
        [--launches gpurun_out/launches.csv] --tag r01 [--peak-gbs 6453.7]

Writes profiles/<tag>_ncu_full.md (one row per captured launch: duration,
DRAM read/write bytes, achieved DRAM GB/s and % of peak, L1 sectors per
global-load request -- the sector efficiency of the block-label gathers --,
L2 hit rate, warps active, registers) and profiles/ncu_summary.json
(per-kernel DRAM bytes per launch, read by bench.py as roofline.traffic).
With --launches also profiles/<tag>_launches.md: per-kernel totals of the
`--metrics gpu__time_duration.sum` launch list (cold-cache, serialised:
compare shares, not absolutes).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "ld_sectors": "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "ld_requests": "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "st_sectors": "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "st_requests": "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
}
TIME = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
BYTES = {"byte": 1.0, "B": 1.0, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9,
         "Tbyte": 1e12, "TB": 1e12}
SCALE = {"dur_us": TIME, "dram_rd": BYTES, "dram_wr": BYTES}


def short(name):
    """Kernel name without namespaces, template arguments and parameters
    (the first identifier ending in `_kernel`)."""
    import re
    for tok in re.findall(r"[A-Za-z_]\w*", name.split("(")[0] if "_kernel(" in name else name):
        if tok.endswith("_kernel"):
            return tok
    return name.split("(")[0]


def read_raw(rep):
    if rep.endswith(".csv"):
        text = open(rep).read()
    else:
        text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                              check=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for key, m in METRICS.items():
            if m not in hdr:
                d[key] = None
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                d[key] = None
                continue
            table = SCALE.get(key)
            if table is not None and units[i] not in table:
                raise ValueError(f"unknown unit {units[i]!r} for {m}")
            d[key] = v * (table[units[i]] if table is not None else 1.0)
        res.append(d)
    return res


def read_launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    agg = OrderedDict()
    total = 0.0
    for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = TIME[r["Metric Unit"]]
        v = float(r["Metric Value"].replace(",", "")) * scale
        name = short(r["Kernel Name"])
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        total += v
    return agg, total


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rep", action="append", default=[],
                   help="ncu report or raw-page CSV; NAME=PATH to label a workload (repeatable)")
    p.add_argument("--launches")
    p.add_argument("--tag", required=True)
    p.add_argument("--note", default="")
    p.add_argument("--peak-gbs", type=float, default=None)
    a = p.parse_args()
    peak = a.peak_gbs
    if peak is None:
        try:
            peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        except Exception:
            peak = 6650.0
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.rep:
        md = [f"# ncu --set full, {a.tag}", "", a.note, "",
              f"DRAM peak for the % column: {peak:.0f} GB/s (MEASURED_PEAKS.json hbm_gbs, of measured).  "
              "`ld sectors/req`: 32-byte L1 sectors per warp-wide global load request (4 = fully coalesced 32-bit "
              "loads; ~32 = every lane in a different sector, i.e. random block-label gathers, whose sector "
              "efficiency is 4 B used of 32 B moved).  `L1 %` / `L2 %`: l1tex / lts throughput as % of peak -- the "
              "gather-bound kernels sit on the L1TEX line rate, not on DRAM.", ""]
        summary = {}
        for spec in a.rep:
            name, path = spec.split("=", 1) if "=" in spec else (os.path.basename(spec), spec)
            rows = read_raw(path)
            md += [f"## {name}", "",
                   "| kernel | us | DRAM rd MB | DRAM wr MB | DRAM GB/s | % of peak | ld sectors/req | st sectors/req "
                   "| L1 % | L2 % | L2 hit % | warps active % | regs |",
                   "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
            for d in rows:
                if not d["dur_us"]:
                    continue
                byts = (d["dram_rd"] or 0) + (d["dram_wr"] or 0)
                gbs = byts / (d["dur_us"] * 1e-6) / 1e9
                spr = d["ld_sectors"] / d["ld_requests"] if d["ld_requests"] else float("nan")
                sspr = d["st_sectors"] / d["st_requests"] if d.get("st_requests") else float("nan")
                md.append(f"| {d['kernel']} | {d['dur_us']:.1f} | {(d['dram_rd'] or 0) / 1e6:.1f} | "
                          f"{(d['dram_wr'] or 0) / 1e6:.1f} | {gbs:.0f} | {100 * gbs / peak:.1f} | {spr:.2f} | "
                          f"{sspr:.2f} | {d['l1_pct'] or 0:.0f} | {d['lts_pct'] or 0:.0f} | {d['l2_hit'] or 0:.1f} | "
                          f"{d['warps'] or 0:.1f} | {int(d['regs'] or 0)} |")
                s_ = summary.setdefault(d["kernel"], {"launches": 0, "dram_bytes": 0.0, "us": 0.0, "workload": name})
                if s_["workload"] != name:
                    continue  # per-launch figures of the first workload that runs the kernel, not a blend
                s_["launches"] += 1
                s_["dram_bytes"] += byts
                s_["us"] += d["dur_us"] or 0
            md.append("")
        for s_ in summary.values():
            s_["dram_bytes_per_launch"] = s_["dram_bytes"] / s_["launches"]
            s_["us_per_launch"] = s_["us"] / s_["launches"]
        with open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu_full.md"), "w") as f:
            f.write("\n".join(md) + "\n")
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
            json.dump({"tag": a.tag, "kernels": summary}, f, indent=1)
    if a.launches:
        agg, total = read_launches(a.launches)
        md = [f"# launch list ({a.tag})", "", a.note, "",
              "`ncu --metrics gpu__time_duration.sum --clock-control none`: every launch serialised and cold-cache, so "
              "compare each kernel's SHARE with the bench's live per-kernel profile, not absolute times.", "",
              "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for name, (cnt, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append(f"| {name} | {cnt} | {us:.1f} | {100 * us / total:.1f}% |")
        with open(os.path.join(ROOT, "profiles", f"{a.tag}_launches.md"), "w") as f:
            f.write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
