"""ncu CSV (--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum) of the
headline step -> profiles/r02_traffic.json (per-kernel DRAM bytes; read by bench.py's roofline).
usage: python tools/traffic_json.py traffic.csv > profiles/r02_traffic.json"""
import csv, json, re, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
iK, iM, iV, iID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
names = {}
for r in rows[start + 1:]:
    if len(r) <= iV:
        continue
    per[r[iID]][r[iM]] = float(r[iV].replace(",", ""))
    names[r[iID]] = r[iK]
KEYS = [("spectrum", r"oaa_spectrum_kernel"), ("xspec", r"oaa_xspec_kernel<8, 0>"), ("walk", r"oaa_walk_kernel<8, 3, 0, 0>"),
        ("bwdd", r"oaa_bwdd_kernel"), ("xspec_win", r"oaa_xspec_kernel<8, 1>"), ("bwdf", r"oaa_bwdf_kernel"),
        ("finalize", r"oaa_filter_finalize_kernel")]
out = {"what": "per-launch DRAM traffic of the headline step's kernels (N=224 n=8 C=3 K=64 B=128, Valid), one ncu "
               "pass with dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum (--clock-control none; "
               "serialized, cold-cache launch times)",
       "command": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none "
                  "--csv python tools/prof_step.py 1",
       "kernels": {}}
for key, pat in KEYS:
    for i, nm in names.items():
        if pat in nm:
            m = per[i]
            rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
            unit = 1e-3 if m.get("gpu__time_duration.sum", 0) > 1e5 else 1e-3
            out["kernels"][key] = {"kernel": nm, "dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
                                   "ncu_ms": m.get("gpu__time_duration.sum", 0.0) * 1e-6}
            break
print(json.dumps(out, indent=1))
