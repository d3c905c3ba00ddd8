"""Summarise an ncu report: key metrics + SASS opcode mix + top stall reasons."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = {"Duration", "Executed Ipc Active", "Registers Per Thread", "Achieved Active Warps Per SM", "L1/TEX Hit Rate",
        "Grid Size", "Block Size", "DRAM Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
        "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "Memory Throughput"}
rows = list(csv.reader(det.splitlines()))
if rows:
    h = rows[0]
    iN, iU, iV = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    for row in rows[1:]:
        if len(row) > iV and row[iN] in want:
            print(f"{row[iN]:40s} {row[iV]} {row[iU]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(raw))
hdr, vals = r[0], r[2]
stalls = []
for h, v in zip(hdr, vals):
    if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
        try: stalls.append((float(v.replace(',', '')), h.split("stalled_")[1]))
        except: pass
    if h in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
             "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"):
        print(f"{h:60s} {v}")
print("top stalls (cycles per issued instr):", ", ".join(f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]; iS = h.index("Source"); iE = h.index("Instructions Executed"); iW = h.index("Warp Stall Sampling (All Samples)")
ex, st = Counter(), Counter(); T = S = 0
for row in rows[2:]:
    try: e = int(row[iE]); s = int(row[iW])
    except: continue
    toks = row[iS].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    ex[op] += e; st[op] += s; T += e; S += s
print("warp-instr", T)
print("  ".join(f"{o}:{100*c/T:.1f}%/{100*st[o]/max(S,1):.0f}%st" for o, c in ex.most_common(18)))
