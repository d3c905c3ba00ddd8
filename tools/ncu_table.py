"""One markdown row per kernel of an ncu report (--set full): duration, DRAM traffic,
issue / pipe utilisation, shared-memory wavefronts, tensor pipe, occupancy.
usage: python tools/ncu_table.py report.ncu-rep [title]"""
import csv, re, subprocess, sys
rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
h, units = raw[0], raw[1]
cols = [("gpu__time_duration.sum", "ms", 1e-6), ("dram__bytes_read.sum", "DRAM rd GB", 1e-9),
        ("dram__bytes_write.sum", "DRAM wr GB", 1e-9), ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue %", 1),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %", 1),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %", 1),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts M", 1e-6),
        ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe %", 1),
        ("smsp__inst_executed.sum", "warp instr M", 1e-6), ("launch__registers_per_thread", "regs", 1),
        ("sm__warps_active.avg.per_cycle_active", "warps/SM", 1)]
def find(name):
    for i, k in enumerate(h):
        if k == name or k.endswith("." + name) or k.split(".", 2)[-1] == name:
            return i
    return None
idx = [(find(c), lab, sc) for c, lab, sc in cols]
iK = h.index("Kernel Name")
out = [f"## {title}", "", "| kernel | " + " | ".join(l for _, l, _ in idx) + " |", "|---" * (len(idx) + 1) + "|"]
for r in raw[2:]:
    name = r[iK]
    m = re.search(r"(oaa_\w+<[^>]*>|oaa_\w+)", name)
    cells = []
    for i, _, sc in idx:
        try:
            v = float(r[i].replace(",", "")) if i is not None else None
        except ValueError:
            v = None
        if v is not None:  # normalise ncu's auto-scaled units to ns / bytes first
            u = units[i]
            v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ms": 1e6, "us": 1e3, "ns": 1, "second": 1e9, "byte": 1, "Kbyte": 1e3,
                  "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            v *= sc
        cells.append("-" if v is None else (f"{v:.3f}" if v < 100 else f"{v:.0f}"))
    out.append(f"| `{m.group(1) if m else name[:40]}` | " + " | ".join(cells) + " |")
print("\n".join(out))
