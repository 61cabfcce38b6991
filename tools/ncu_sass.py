"""Top SASS instructions of one kernel by stall samples, with their dominant
stall reasons: python tools/ncu_sass.py REPORT KERNEL_REGEX [N] [launch_skip]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source=sass", "-s", skip, "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
recs = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    st = sorted(((float(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    recs.append((s, r[ix["Address"]], r[ix["Source"]], st))
tot = sum(x[0] for x in recs) or 1
byreason = {}
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    for h in stalls:
        try:
            byreason[h[6:]] = byreason.get(h[6:], 0) + float(r[ix[h]] or 0)
        except ValueError:
            pass
print("total samples", tot, {k: round(100 * v / tot, 1) for k, v in sorted(byreason.items(), key=lambda kv: -kv[1])[:8]})
for s, a, src, st in sorted(recs, key=lambda x: -x[0])[:N]:
    print(f"{100*s/tot:5.1f}% {a:>6} {src[:60]:60s} " + " ".join(f"{n}:{int(v)}" for v, n in st if v))
