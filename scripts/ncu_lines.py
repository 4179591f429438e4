#!/usr/bin/env python3
"""Per-source-line executed warp instructions and stall samples of one ncu capture (needs -lineinfo):
  python scripts/ncu_lines.py <report.ncu-rep> [top]"""
import csv
import subprocess
import sys


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if "Instructions Executed" in r)
    i_ie, i_s = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    num = lambda v: int(v) if v and v.lstrip("-").isdigit() else 0
    lines = {}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= i_ie or not r[0] or not r[0].isdigit():
            continue
        lines[(int(r[0]), r[1][:100])] = [num(r[i_ie]), num(r[i_s])]
    tot = sum(v[0] for v in lines.values()) or 1
    ts = sum(v[1] for v in lines.values()) or 1
    print(f"total warp instructions {tot}, stall samples {ts}")
    for k, v in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]:
        print("%5.1f%% inst %5.1f%% stall  L%-4d %s" % (100 * v[0] / tot, 100 * v[1] / ts, k[0], k[1].strip()))


if __name__ == "__main__":
    main()
