"""Top stalled SASS instructions of one kernel in an ncu report:
python tools/ncu_hot.py REPORT KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source=sass", "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
data = []
for r in rows:
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
val = lambda r: int(r[i_s]) if r[i_s].isdigit() else 0
tot = sum(val(r) for r in data)
print("total samples", tot, "sass lines", len(data))
for r in sorted(data, key=lambda r: -val(r))[:N]:
    print(f"{val(r):6d} {100.0*val(r)/max(tot,1):5.1f}% {r[0]:>6} {r[i_src][:100]}")
