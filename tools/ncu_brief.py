#!/usr/bin/env python
"""Key metrics and top stall reasons per launch from `ncu --page raw --csv`.

    python tools/ncu_brief.py RAW.csv [launch-index ...]
"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units, data = rows[0], rows[1], rows[2:]
    sel = [int(x) for x in sys.argv[2:]] or range(len(data))
    for i in sel:
        r = data[i]
        print(f"[{i}] {r[hdr.index('Kernel Name')][:80]}")
        for k in KEYS:
            if k in hdr:
                print(f"    {k:58s} {r[hdr.index(k)]} {units[hdr.index(k)]}")
        st = [(h[len('smsp__pcsamp_warps_issue_stalled_'):], float(r[j] or 0)) for j, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1
        print("    stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for n, v in sorted(st, key=lambda x: -x[1])[:7]))


if __name__ == "__main__":
    main()
