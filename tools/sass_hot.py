"""Group the SASS of an ncu report by execution count (≈ which loop level) and show the
instruction mix of each group: python tools/sass_hot.py report.ncu-rep"""
import csv, subprocess, sys
from collections import Counter, defaultdict
src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]; iS = h.index("Source"); iE = h.index("Instructions Executed"); iW = h.index("Warp Stall Sampling (All Samples)")
groups = defaultdict(lambda: [0, 0, Counter(), 0])
E = S = 0
for r in rows[2:]:
    try: e = int(r[iE]); w = int(r[iW])
    except (ValueError, IndexError): continue
    if e == 0: continue
    t = r[iS].split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    k = float(f"{e:.2g}")
    g = groups[k]; g[0] += e; g[1] += w; g[2][op] += e; g[3] += 1
    E += e; S += w
for k, (e, w, ops, n) in sorted(groups.items(), key=lambda kv: -kv[1][0])[:10]:
    print(f"count~{k:.2g} ({n} instrs): {100*e/E:5.1f}% of instr, {100*w/S:5.1f}% of stalls | " +
          " ".join(f"{o}:{c//int(k) if k else 0}" for o, c in ops.most_common(10)))
