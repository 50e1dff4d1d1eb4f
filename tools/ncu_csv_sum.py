"""Summarise an ncu --csv --metrics log: per kernel name, launches and the sum of every metric
(measurement tool).  usage: ncu_csv_sum.py log.csv [skip_first_n_launches]"""
import csv
import sys

path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
agg, seen = {}, {}
for r in rows[1:]:
    lid = int(r[ii])
    if lid < skip:
        continue
    k = r[ki].split("(")[0].replace("void ", "")
    a = agg.setdefault(k, {})
    a[r[mi]] = a.get(r[mi], 0.0) + float(r[vi].replace(",", ""))
    seen.setdefault(k, set()).add(lid)
tot = {}
for k, a in sorted(agg.items(), key=lambda x: -x[1].get("gpu__time_duration.sum", 0)):
    print(f"{k[:58]:58s} launches {len(seen[k]):5d}")
    for m, v in a.items():
        print(f"    {m:70s} {v:.6g}")
        tot[m] = tot.get(m, 0) + v
print("TOTAL")
for m, v in tot.items():
    print(f"    {m:70s} {v:.6g}")
