"""Per-CUDA-source-line stall samples and instruction counts from an ncu report
(the first kernel of the report; capture one kernel per report).
usage: ncu_lines.py REPORT [TOP]"""
import csv
import io
import os
import subprocess
import sys


def main(path, top=40):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    hdr, fname, agg = None, "?", []
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0] or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        try:
            agg.append((float(d["Warp Stall Sampling (All Samples)"]), float(d["Instructions Executed"]),
                        f"{fname}:{r[0]}", r[1].strip()[:95]))
        except (ValueError, KeyError):
            pass
    ts = sum(a[0] for a in agg) or 1
    ti = sum(a[1] for a in agg) or 1
    print(f"total samples {ts:.0f}  instructions {ti:.3e}")
    for s, i, ln, src in sorted(agg, reverse=True)[:top]:
        print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% inst  {ln:>22s}: {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
