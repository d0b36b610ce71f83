"""Sum an ncu launch list (gpu__time_duration.sum CSV) per path run: a run starts at the
first kernel after a weighting/finalize kernel.  usage: python tools/sum_launches.py f.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
ki, vi = rows[h].index("Kernel Name"), rows[h].index("Metric Value")
runs, cur, prev_end = [], [], False
for r in rows[h + 1:]:
    name, ns = r[ki], float(r[vi].replace(",", ""))
    if prev_end and not name.startswith("void finalize_split"):
        runs.append(cur)
        cur = []
    cur.append((name.split("(")[0].replace("void ", "").replace("unnamed>::", ""), ns))
    prev_end = name.startswith("void interp") or name.startswith("void finalize_split")
runs.append(cur)
for run in runs:
    tot = sum(ns for _, ns in run)
    print(f"total {tot / 1e3:8.1f} us  " + "  ".join(f"{n[:28]}={ns / 1e3:.1f}" for n, ns in run))
