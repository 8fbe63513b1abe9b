"""Per-CUDA-source-line instruction and stall totals of an ncu --set full
report captured with --import-source on (compile with -lineinfo).

    python tools/ncu_lines.py rep.ncu-rep [--file stream_codec.cu] [--top 40]
"""
import argparse
import csv
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--file", default="")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda"],
                         capture_output=True, text=True).stdout
    hdr, rows, name = None, [], None
    out = []
    for r in csv.reader(txt.splitlines()):
        if not r:
            continue
        if r[0] == "Kernel Name":
            if hdr and rows:
                out.append((name, hdr, rows))
            name, hdr, rows = r[1], None, []
        elif r[0] in ("#", "Line", "Line #"):
            hdr = r
        elif hdr and len(r) == len(hdr):
            rows.append(r)
    if hdr and rows:
        out.append((name, hdr, rows))
    for name, hdr, rows in out:
        print(f"=== {name[:100]}")
        print("    columns:", [h for h in hdr][:12])
        i_src = hdr.index("Source")
        i_ex = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else None
        i_st = hdr.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in hdr else None
        i_ln = 0
        tot = sum(float(r[i_ex] or 0) for r in rows) or 1.0
        stot = sum(float(r[i_st] or 0) for r in rows) if i_st is not None else 1.0
        top = sorted(rows, key=lambda r: -float(r[i_ex] or 0))[: a.top]
        for r in top:
            ex = float(r[i_ex] or 0)
            st = float(r[i_st] or 0) if i_st is not None else 0
            print(f"{ex / tot * 100:6.2f}% inst {st / stot * 100:6.2f}% stall  L{r[i_ln]:>5}  {r[i_src].strip()[:110]}")


if __name__ == "__main__":
    main()
