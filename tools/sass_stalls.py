"""Per-instruction stall breakdown from an ncu source-page CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], []
for r in rows[2:]:  # first kernel only (a capture of several repeats the header)
    if r and r[0] in ("Kernel Name", "Address"):
        break
    data.append(r)
col = {h: i for i, h in enumerate(hdr)}
reasons = ["stall_long_sb", "stall_wait", "stall_short_sb", "stall_branch_resolving", "stall_membar", "stall_lg",
           "stall_mio", "stall_math", "stall_sleep", "stall_selected", "stall_not_selected", "stall_no_inst"]
f = lambda r, k: float(r[col[k]] or 0)  # noqa: E731
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
agg = {k: sum(f(r, k) for r in data) for k in reasons}
print("totals:", {k[6:]: round(v / tot * 100, 1) for k, v in agg.items()})
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for k in ("stall_long_sb", "stall_wait", "stall_short_sb"):
    print(f"--- top {k}")
    idx = sorted(range(len(data)), key=lambda i: -f(data[i], k))[:top // 3]
    for i in sorted(idx):
        r = data[i]
        print(f"{i:5d} {f(r, k) / tot * 100:5.2f}% ex={r[col['Instructions Executed']]:>8} {r[col['Source']][:80]}")
