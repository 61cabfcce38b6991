"""Markdown summary of an `ncu --set full` report: per kernel the duration,
DRAM traffic, occupancy limits, issue activity, FP64 pipe use and the top
stall reasons.

    python tools/ncu_summary.py REPORT.ncu-rep > profiles/rNN_..._ncu_full.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("time", "gpu__time_duration.sum", 1),
    ("DRAM read MB", "dram__bytes_read.sum", None),
    ("DRAM write MB", "dram__bytes_write.sum", None),
    ("regs", "launch__registers_per_thread", 1),
    ("block", "launch__block_size", 1),
    ("grid", "launch__grid_size", 1),
    ("CTA/SM (regs)", "launch__occupancy_limit_registers", 1),
    ("CTA/SM (smem)", "launch__occupancy_limit_shared_mem", 1),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("FP64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("warp instr (M)", "smsp__inst_executed.sum", 1e-6),
    ("smem bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
]


def to_mb(v, unit):
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
    return v * scale


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full summary: {sys.argv[1]}\n")
    names = [d[col["Kernel Name"]].split("(")[0] for d in data]
    print("| metric | " + " | ".join(names) + " |")
    print("|---|" + "---|" * len(names))
    for label, m, sc in METRICS:
        if m not in col:
            continue
        vals = []
        for d in data:
            raw = d[col[m]].replace(",", "")
            try:
                v = float(raw)
            except ValueError:
                vals.append(raw)
                continue
            v = to_mb(v, units[col[m]]) if sc is None else v * sc
            vals.append(f"{v:.3g}" if abs(v) < 1e4 else f"{v:.0f}")
        unit = units[col[m]] if sc == 1 and label == "time" else ""
        print(f"| {label}{' (' + unit + ')' if unit else ''} | " + " | ".join(vals) + " |")
    st = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
          and h.endswith("_per_issue_active.ratio")]
    print("\nTop stall reasons (warps stalled per issued instruction):\n")
    for d, nm in zip(data, names):
        vals = sorted(((float(d[col[h]] or 0), h[len("smsp__average_warps_issue_stalled_"):-len(
            "_per_issue_active.ratio")]) for h in st), reverse=True)[:5]
        print(f"- {nm}: " + ", ".join(f"{n} {v:.2f}" for v, n in vals))


if __name__ == "__main__":
    main()
