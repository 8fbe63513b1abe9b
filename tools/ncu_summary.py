"""Summarise an ncu --set full report: key raw metrics, stall reasons and the
SASS op mix of every profiled kernel.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--ops 16] [--top 8]
"""
import argparse
import collections
import csv
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]


def raw_pages(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    return h, rows[2:]


def source_sections(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    sections, cur = [], None
    for r in csv.reader(txt.splitlines()):
        if not r:
            continue
        if r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            sections.append(cur)
        elif r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
            cur["rows"].append(r)
    return sections


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--ops", type=int, default=16)
    ap.add_argument("--top", type=int, default=8)
    a = ap.parse_args()
    h, rows = raw_pages(a.rep)
    secs = source_sections(a.rep)
    for k, v in enumerate(rows):
        get = lambda n: v[h.index(n)] if n in h else "?"  # noqa: E731
        print(f"=== launch {k}: {get('Kernel Name')[:110]}")
        for n in KEYS:
            print(f"{get(n):>18} {n}")
        st = {h[i]: float(v[i]) for i in range(len(h))
              if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued")
              and v[i].replace('.', '', 1).isdigit()}
        tot = sum(st.values()) or 1.0
        for n, x in sorted(st.items(), key=lambda t: -t[1])[:8]:
            print(f"  {x / tot * 100:5.1f}% {n.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
    for s in secs:
        hh = s["hdr"]
        i_src, i_ex = hh.index("Source"), hh.index("Instructions Executed")
        i_th = hh.index("Thread Instructions Executed")
        i_s = hh.index("Warp Stall Sampling (All Samples)")
        c, ct, sc = collections.Counter(), collections.Counter(), collections.Counter()
        for r in s["rows"]:
            toks = r[i_src].strip().split()
            if not toks:
                continue
            op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
            c[op] += float(r[i_ex] or 0)
            ct[op] += float(r[i_th] or 0)
            sc[op] += float(r[i_s] or 0)
        t, S = sum(c.values()) or 1.0, sum(sc.values()) or 1.0
        print(f"--- SASS mix: {s['name'][:110]}  (warp inst {t:.3g}, thread inst {sum(ct.values()):.3g})")
        for op, n in c.most_common(a.ops):
            print(f"    {op:10s} {n / t * 100:5.1f}%  thr {ct[op]:.3g}  stall {sc[op] / S * 100:5.1f}%")
        top = sorted(s["rows"], key=lambda r: -float(r[i_s] or 0))[:a.top]
        print("  top stall instructions:")
        for r in top:
            print(f"    {float(r[i_s]) / S * 100:5.1f}%  {r[i_src].strip()[:80]}")


if __name__ == "__main__":
    main()
