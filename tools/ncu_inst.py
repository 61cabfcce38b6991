"""Per-CUDA-line executed warp instructions of one kernel (instruction-count
hot spots): python tools/ncu_inst.py REPORT KERNEL_REGEX [N] [launch_skip]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source=cuda,sass", "-s", skip, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
recs, cur, hdr = [], None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split('/')[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            inst = float(r[7])
        except ValueError:
            inst = 0
        recs.append((inst, cur, r[0], r[1][:90]))
tot = sum(x[0] for x in recs) or 1
print(f"warp-instructions {tot:.0f}")
for x in sorted(recs, reverse=True)[:N]:
    print(f"{100*x[0]/tot:5.1f}% {x[1]}:{x[2]} {x[3]}")
