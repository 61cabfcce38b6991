"""Per-CUDA-source-line instructions executed and stall samples of one kernel:
python tools/ncu_lines.py REPORT KERNEL_REGEX [N] [launch_skip]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source=cuda,sass", "-s", skip, "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = None
recs = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        def num(i):
            try:
                return float(r[i])
            except ValueError:
                return 0.0
        recs.append((cur, int(r[0]), num(4), num(7), r[1][:80]))
ts = sum(x[2] for x in recs) or 1
ti = sum(x[3] for x in recs) or 1
print(f"samples {ts:.0f} warp-instructions {ti:.0f}")
for f, ln, s, i, src in sorted(recs, key=lambda x: -x[2])[:N]:
    print(f"{100*s/ts:5.1f}% samp {100*i/ti:5.1f}% inst  {f}:{ln}  {src}")
