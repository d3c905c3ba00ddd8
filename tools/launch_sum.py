"""Per-kernel mean duration from an `ncu --metrics gpu__time_duration.sum --csv` launch list.
usage: python tools/launch_sum.py launches.csv"""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]; iK = h.index("Kernel Name"); iV = h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    try: agg[r[iK].split('(')[0][:60]].append(float(r[iV].replace(',', '')) / 1e6)
    except ValueError: pass
for k, v in agg.items():
    print(f"  {k:60s} n={len(v):4d} mean={sum(v)/len(v):8.3f} ms")
