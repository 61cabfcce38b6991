"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
the kernels in an `ncu --set full` capture of tools/prof_case.py (one
full, low and high product), keyed like bench.py's per-kernel table
("full:k_mid", ...):

    python tools/ncu_traffic.py REPORT.ncu-rep > profiles/rNN_traffic.json
"""
import csv
import io
import json
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ki = hdr.index("Kernel Name")
ri, wi = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
ti = hdr.index("gpu__time_duration.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
res, order, mode = {}, ["full", "low", "high"], -1
prev = None
for r in rows[2:]:
    name = r[ki]
    base = re.sub(r"^void ", "", name).replace("<unnamed>::", "").replace("unnamed>::", "").replace("(anonymous namespace)::", "").split("(")[0]
    base = re.sub(r"^(\w+::)*", "", base.split("<")[0]) if "<" in base else re.sub(r"^(\w+::)*", "", base)
    if base in ("k_zstat", "k_zsplit") or (base == "k_zgen_t" and prev != "k_zstat"):
        mode += 1
    prev = base
    short = {"k_zgen_t": "k_zgen", "k_f1d_ct": "k_f1", "k_f1_ct": "k_f1", "k_f1_pp": "k_f1", "k_ilast_ct": "k_ilast",
             "k_ilast_pp": "k_ilast", "k_mid_4096": "k_mid"}.get(base, base)
    by = float(r[ri]) * scale.get(units[ri], 1) + float(r[wi]) * scale.get(units[wi], 1)
    res[f"{order[mode % 3]}:{short}"] = {"dram_bytes": by, "kernel": name, "us": float(r[ti])}
json.dump({"source": sys.argv[1], "per_launch": res}, sys.stdout, indent=1)
print()
