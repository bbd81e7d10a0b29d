"""Summarise ncu captures into profiles/<round>_*.md / .csv.

  python profiles/summarize.py <round> gpurun_out/launches.csv gpurun_out/prof.ncu-rep [...]

launches.csv: `ncu --metrics gpu__time_duration.sum --clock-control none --csv` launch list
(cold-cache, serialised: compare shares, not absolutes).  *.ncu-rep: `--set full` captures.
"""
import csv
import io
import os
import re
import subprocess
import sys
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("lts__t_requests_srcunit_tex_op_atom_dot_alu.sum", "L2 atom requests"),
    ("lts__t_requests_srcunit_tex_op_atom_dot_cas.sum", "L2 CAS requests"),
    ("lts__t_requests_srcunit_tex_op_red.sum", "L2 red requests"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[idx["Kernel Name"]])[:70]
        v = float(r[idx["Metric Value"]].replace(",", ""))
        u = r[idx["Metric Unit"]]
        v = v / 1000 if u == "ns" else (v * 1000 if u == "ms" else v)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    out = ["| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f} % |")
    return "\n".join(out)


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        kname = d['Kernel Name'].split('(')[0]
        out.append(f"#### `{kname}` (grid {d.get('launch__grid_size', '?')} x {d.get('launch__block_size', '?')})")
        out.append("| metric | value |")
        out.append("|---|---|")
        for k, label in KEYS:
            if k in d:
                out.append(f"| {label} (`{k}`) | {d[k]} {u.get(k, '')} |")
        st = sorted(((k, float(v)) for k, v in d.items()
                     if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio", k) and v),
                    key=lambda x: -x[1])[:6]
        out.append("| top stall reasons (warps per issue) | " +
                   ", ".join(f"{k.split('stalled_')[1].split('_per')[0]} {v:.1f}" for k, v in st) + " |")
        out.append("")
    return "\n".join(out)


def main():
    rnd = sys.argv[1]
    parts = [f"# ncu summary, {rnd}\n"]
    for p in sys.argv[2:]:
        if p.endswith(".csv"):
            parts.append(f"## Launch list (`{os.path.basename(p)}`; cold-cache, serialised — compare shares)\n")
            parts.append(launches(p) + "\n")
        else:
            parts.append(f"## Full capture `{os.path.basename(p)}`\n")
            parts.append(full(p) + "\n")
    path = os.path.join(HERE, f"{rnd}_ncu_summary.md")
    open(path, "w").write("\n".join(parts))
    print(path)


if __name__ == "__main__":
    main()
