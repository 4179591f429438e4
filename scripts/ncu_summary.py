#!/usr/bin/env python3
"""Summarise ncu output for profiles/ (run here, on the CPU box, after gpurun brings it back).

  python scripts/ncu_summary.py full   <report.ncu-rep> <out-prefix> [--candidates N]
  python scripts/ncu_summary.py launches <launches.csv> <out-prefix>

`full` writes <prefix>.md (+ .json) with DRAM bytes, issue / pipe utilisation, occupancy, top stall
reasons and the executed-instruction mix; with --candidates it also writes the per-launch DRAM
traffic that bench.py reports as roofline.traffic. `launches` sums gpu__time_duration per kernel.
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread", "launch__block_size",
    "launch__grid_size", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def full(rep, prefix, candidates=None):
    rows = ncu_csv(["-i", rep, "--page", "raw"])
    hdr, units, val = rows[0], rows[1], rows[2]
    kname = val[hdr.index("Kernel Name")]
    m = {k: (val[hdr.index(k)], units[hdr.index(k)]) for k in KEYS if k in hdr}
    stalls = sorted(((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(val[i] or 0)) for i, h in enumerate(hdr)
                     if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")),
                    key=lambda x: -x[1])
    tot = sum(v for _, v in stalls) or 1.0
    src = ncu_csv(["-i", rep, "--page", "source", "--print-source=sass"])
    sh = src[1]
    si, ei = sh.index("Source"), sh.index("Instructions Executed")
    mix = collections.Counter()
    for r in src[2:]:
        if len(r) <= ei or not r[ei]:
            continue
        toks = r[si].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        mix[op.split(".")[0]] += int(r[ei])
    itot = sum(mix.values()) or 1
    rd = float(m["dram__bytes_read.sum"][0]) * (1e6 if m["dram__bytes_read.sum"][1] == "Mbyte" else 1e9 if m["dram__bytes_read.sum"][1] == "Gbyte" else 1)
    wr = float(m["dram__bytes_write.sum"][0]) * (1e6 if m["dram__bytes_write.sum"][1] == "Mbyte" else 1e9 if m["dram__bytes_write.sum"][1] == "Gbyte" else 1)
    js = {"kernel": kname, "metrics": {k: v[0] + " " + v[1] for k, v in m.items()},
          "stalls_pct": {k: round(100 * v / tot, 1) for k, v in stalls[:10]},
          "inst_mix_pct": {k: round(100 * v / itot, 1) for k, v in mix.most_common(15)},
          "dram_bytes_per_launch": rd + wr}
    if candidates:
        js["candidates_per_launch"] = candidates
        js["dram_bytes_per_candidate"] = (rd + wr) / candidates
        js["warp_inst_per_candidate"] = float(m["smsp__inst_executed.sum"][0]) / candidates
    with open(prefix + ".json", "w") as f:
        json.dump(js, f, indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"# ncu --set full: `{kname}`\n\nSource report: `{rep}`\n\n| metric | value |\n|---|---|\n")
        for k, v in m.items():
            f.write(f"| {k} | {v[0]} {v[1]} |\n")
        if candidates:
            f.write(f"| candidates per launch | {candidates} |\n| DRAM bytes per candidate | {js['dram_bytes_per_candidate']:.0f} |\n"
                    f"| warp instructions per candidate | {js['warp_inst_per_candidate']:.0f} |\n")
        f.write("\n## Warp stall reasons (share of samples)\n\n")
        for k, v in stalls[:10]:
            f.write(f"- {k}: {100 * v / tot:.1f}%\n")
        f.write("\n## Executed instruction mix\n\n")
        for k, v in mix.most_common(15):
            f.write(f"- {k}: {100 * v / itot:.1f}%\n")
    print(json.dumps(js, indent=1))


def launches(path, prefix):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = collections.OrderedDict()
    for r in rows[1:]:
        ns = float(r[vi].replace(",", "")) * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r[ui], 1)
        per.setdefault(r[ki], []).append(ns)
    tot = sum(sum(v) for v in per.values())
    with open(prefix + ".md", "w") as f:
        f.write(f"# ncu launch list (`gpu__time_duration.sum`, --clock-control none)\n\nSource: `{path}`\n\n"
                "Cold-cache, serialised per-launch times: compare SHARES, not absolutes.\n\n"
                "| kernel | launches | total ms | mean ms | share |\n|---|---|---|---|---|\n")
        for k, v in per.items():
            f.write(f"| `{k[:70]}` | {len(v)} | {sum(v) / 1e6:.3f} | {sum(v) / len(v) / 1e6:.3f} | {100 * sum(v) / tot:.1f}% |\n")
    print(open(prefix + ".md").read())


if __name__ == "__main__":
    if sys.argv[1] == "full":
        cands = int(sys.argv[sys.argv.index("--candidates") + 1]) if "--candidates" in sys.argv else None
        full(sys.argv[2], sys.argv[3], cands)
    else:
        launches(sys.argv[2], sys.argv[3])
