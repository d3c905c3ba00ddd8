"""Aggregate executed instructions and stall samples by CUDA source line (ncu report
imported with --import-source on).  usage: python tools/src_lines.py report [file-substring] [top]"""
import csv, subprocess, sys
rep = sys.argv[1]; sub = sys.argv[2] if len(sys.argv) > 2 else ""; top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res = []; fname = None; h = None
for r in rows:
    if len(r) == 2 and r[0] == "File Name": fname = r[1]; h = None; continue
    if r and r[0] == "Line No" or (r and "Instructions Executed" in r): h = r; continue
    if h is None or len(r) != len(h): continue
    d = dict(zip(h, r))
    try: e = int(d.get("Instructions Executed", "0") or 0); w = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError: continue
    if e == 0 and w == 0: continue
    if sub and sub not in (fname or ""): continue
    res.append((e, w, (fname or "").split("/")[-1], d.get("Line No", d.get("#", "?")), d.get("Source", "")[:90]))
E = sum(x[0] for x in res) or 1; W = sum(x[1] for x in res) or 1
for e, w, f, l, s in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{100*e/E:5.1f}% inst {100*w/W:5.1f}% stall  {f}:{l}  {s.strip()}")
