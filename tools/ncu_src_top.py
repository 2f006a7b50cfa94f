#!/usr/bin/env python
"""Top source lines of one kernel by warp-stall samples and executed
instructions, from `ncu -i REP --page source --csv --print-source cuda,sass`.

    python tools/ncu_src_top.py SRC.csv [N]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hdr = next(r for r in rows if r and r[0] == "Line No")
    i_samp = hdr.index("Warp Stall Sampling (All Samples)")
    i_inst = hdr.index("Instructions Executed")
    lines = []
    for r in rows:
        if len(r) > i_inst and r[0] not in ("", "Line No") and r[0].isdigit():
            try:
                lines.append((int(r[i_samp] or 0), int(r[i_inst] or 0), int(r[0]), r[1].strip()))
            except ValueError:
                pass
    tot_s = sum(x[0] for x in lines) or 1
    tot_i = sum(x[1] for x in lines) or 1
    print(f"samples {tot_s}, warp instructions {tot_i}")
    for s, i, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"{100 * s / tot_s:5.1f}% stall {100 * i / tot_i:5.1f}% inst  l.{ln:<5d} {src[:110]}")


if __name__ == "__main__":
    main()
