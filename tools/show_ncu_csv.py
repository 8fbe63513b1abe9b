"""Print metric values from `ncu --csv` launch lists: python tools/show_ncu_csv.py file.csv..."""
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows:
        print(f, "no rows")
        continue
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    for r in rows[1:]:
        print(f.split("/")[-1], r[ii], r[ki][:48], r[mi], r[vi])
