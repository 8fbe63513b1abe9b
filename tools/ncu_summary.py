import csv, sys, subprocess, collections
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
get = lambda n: v[h.index(n)] if n in h else "?"
for n in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
          "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]:
    print(f"{get(n):>16} {n}")
st = {h[i]: float(v[i]) for i in range(len(h)) if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued") and v[i].replace('.','',1).isdigit()}
tot = sum(st.values())
for k, x in sorted(st.items(), key=lambda t: -t[1])[:8]:
    print(f"  {x/tot*100:5.1f}% {k.replace('smsp__pcsamp_warps_issue_stalled_','')}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(sass.splitlines()))[1:]
hh = rows[0]; data = rows[1:]
i_src = hh.index("Source"); i_ex = hh.index("Instructions Executed"); i_s = hh.index("Warp Stall Sampling (All Samples)")
c = collections.Counter(); sc = collections.Counter(); t = 0
for r in data:
    toks = r[i_src].strip().split()
    if not toks: continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    n = float(r[i_ex] or 0); c[op] += n; t += n; sc[op] += float(r[i_s] or 0)
S = sum(sc.values())
print("  top ops (share of inst, share of stall samples):")
for op, n in c.most_common(14):
    print(f"    {op:8s} {n/t*100:5.1f}%  stall {sc[op]/S*100:5.1f}%")
top = sorted(data, key=lambda r: -float(r[i_s] or 0))[:8]
print("  top stall instructions:")
for r in top:
    print(f"    {float(r[i_s])/S*100:5.1f}%  {r[i_src].strip()[:70]}")
