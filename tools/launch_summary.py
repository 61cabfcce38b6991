"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into
per-kernel shares of the product step.

    python tools/launch_summary.py LAUNCHES.csv > profiles/rNN_launch_summary.md

Products are the runs of tmg:: kernels that start at the split (k_zsplit,
k_zgen, or k_zstat where the split's carry aggregates are a kernel of their own); bench.py issues them as full, low, high per step (high is
the run containing k_high_round).
"""
import collections
import csv
import statistics
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    def norm(name):
        # "void tmg::<unnamed>::k_carry_lanes<5>(tmg::CarryArgs)" -> "k_carry_lanes<5>"
        name = name.split("(")[0]
        if name.startswith("void "):
            name = name[5:]
        return name.replace("tmg::", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")

    seq = [(norm(r[ki]), float(r[vi].replace(",", "")) / 1e3)
           for r in data if r[mi] == "gpu__time_duration.sum"]
    other = [t for k, t in seq if not k.startswith("k_")]
    groups, cur = [], []
    prev = None
    for k, t in seq:
        if not k.startswith("k_"):
            continue
        starts = k in ("k_zstat", "k_small_product", "k_basecase") or ((k.startswith("k_zgen") or k.startswith("k_zsplit")) and prev != "k_zstat")
        if starts and cur:
            groups.append(cur)
            cur = []
        cur.append((k, t))
        prev = k
    if cur:
        groups.append(cur)
    per = collections.defaultdict(list)
    order = ("full", "low", "high")
    idx = 0
    for g in groups:
        names = [k for k, _ in g]
        mode = "high" if "k_high_round" in names else order[idx % 3]
        idx = idx + 1 if mode != "high" else 0
        for k, t in g:
            per[(mode, k)].append(t)
    tot = {m: sum(statistics.median(v) for (mm, _), v in per.items() if mm == m) for m in order}
    print(f"# ncu launch list summary: {sys.argv[1]}\n")
    print("Cold-cache, serialised per-launch times (`--metrics gpu__time_duration.sum "
          "--clock-control none`); compare shares, not absolutes.\n")
    print("| mode | kernel | launches | median us | share of product |")
    print("|---|---|---|---|---|")
    for m in order:
        for (mm, k), v in per.items():
            if mm == m:
                print(f"| {m} | {k} | {len(v)} | {statistics.median(v):.1f} | "
                      f"{100 * statistics.median(v) / tot[m]:.1f}% |")
        print(f"| {m} | **total** | | {tot[m]:.1f} | 100% |")
    print(f"\nnon-tmg launches (torch fills / L2 flush): {len(other)}, {sum(other):.1f} us total")


if __name__ == "__main__":
    main()
