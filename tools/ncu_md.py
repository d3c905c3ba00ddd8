"""Markdown summary of one `ncu --set full` report (key throughput, occupancy, traffic,
pipe utilisation, stall reasons, instruction mix).  usage: ncu_md.py report title"""
import csv, subprocess, sys
from collections import Counter
rep, title = sys.argv[1], sys.argv[2]
def page(p, extra=()):
    return subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
det = list(csv.reader(page("details").splitlines()))
h = det[0]; iN, iU, iV = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
kname = det[1][h.index("Kernel Name")]
want = ["Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Achieved Active Warps Per SM", "Theoretical Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate"]
vals = {}
for r in det[1:]:
    if len(r) > iV and r[iN] in want and r[iN] not in vals:
        vals[r[iN]] = f"{r[iV]} {r[iU]}".strip()
raw = list(csv.reader(page("raw").splitlines()))
rh, ru, rv = raw[0], raw[1], raw[2]
R = dict(zip(rh, zip(rv, ru)))
def g(k):
    v = R.get(k, ("n/a", ""))
    return f"{v[0]} {v[1]}".strip()
stalls = []
for k, (v, u) in R.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try: stalls.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError: pass
S = sum(x for x, _ in stalls) or 1
src = list(csv.reader(page("source", ("--print-source", "sass")).splitlines()))
sh = src[1]; iS = sh.index("Source"); iE = sh.index("Instructions Executed")
ex = Counter(); T = 0
for r in src[2:]:
    try: e = int(r[iE])
    except (ValueError, IndexError): continue
    t = r[iS].split()
    if not t: continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ex[op] += e; T += e
out = [f"## {title}", "", f"Kernel: `{kname}`", "", "| metric | value |", "|---|---|"]
out += [f"| {k} | {vals[k]} |" for k in want if k in vals]
for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]:
    out.append(f"| `{k}` | {g(k)} |")
out += ["", "Stall reasons (share of warp samples): " + ", ".join(f"{n} {100*x/S:.1f}%" for x, n in sorted(stalls, reverse=True)[:8]), "",
        "SASS instruction mix (share of executed warp instructions): " + ", ".join(f"{o} {100*c/T:.1f}%" for o, c in ex.most_common(14)), ""]
print("\n".join(out))
