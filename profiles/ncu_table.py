"""Key counters of `ncu --set full` captures exported with `ncu -i X --page raw --csv`.
python profiles/ncu_table.py gpurun_out/prof_r2a/*.raw.csv"""
import csv
import os
import sys

KEYS = [("gpu__time_duration.sum", "us", 1), ("smsp__inst_executed.sum", "Minst", 1e-6),
        ("lts__t_requests_srcunit_tex_op_atom_dot_alu.sum", "atom", 1),
        ("lts__t_requests_srcunit_tex_op_atom_dot_cas.sum", "cas", 1),
        ("lts__t_requests_srcunit_tex_op_red.sum", "red", 1),
        ("lts__t_sectors_srcunit_tex_op_read.sum", "rd sect", 1),
        ("lts__t_sectors_srcunit_tex_op_write.sum", "wr sect", 1),
        ("dram__bytes_read.sum", "dram rd MB", None), ("dram__bytes_write.sum", "dram wr MB", None),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ %", 1),
        ("launch__registers_per_thread", "regs", 1)]
STALLS = ["long_scoreboard", "wait", "branch_resolving", "barrier", "math_pipe_throttle", "not_selected",
          "short_scoreboard", "sleeping", "membar", "lg_throttle", "mio_throttle", "no_instruction"]


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def num(d, k, scale):
    if k not in d:
        return float("nan")
    u, v = d[k]
    x = float(v.replace(",", ""))
    if scale is None:  # bytes -> MB
        x *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1e-6)
        return x
    if k == "gpu__time_duration.sum":
        x *= {"ns": 1e-3, "us": 1, "ms": 1e3}.get(u, 1)
    return x * scale


def main(paths):
    print("| capture | " + " | ".join(n for _, n, _ in KEYS) + " | top stalls (warps per issue) |")
    print("|---" * (len(KEYS) + 2) + "|")
    for p in paths:
        d = load(p)
        cells = [f"{num(d, k, s):.4g}" for k, _, s in KEYS]
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in d:
                st.append((float(d[k][1]), s))
        top = ", ".join(f"{s} {v:.1f}" for v, s in sorted(st, reverse=True)[:3])
        print(f"| {os.path.basename(p).replace('.raw.csv', '')} | " + " | ".join(cells) + f" | {top} |")


if __name__ == "__main__":
    main(sys.argv[1:])
