"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(d["Metric Unit"], 1.0)
                out.append((int(d["ID"]), d["Kernel Name"], v * scale))
    return out


def main(path):
    out = load(path)
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for _, n, ms in out:
        k = n.split("(")[0]
        tot[k] += ms
        cnt[k] += 1
    s = sum(tot.values())
    print(f"{len(out)} launches, {s:.1f} ms total (serialised, cold)")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"  {v:10.1f} ms  {100 * v / s:5.1f}%  x{cnt[k]:4d}  {k}")
    return out


if __name__ == "__main__":
    main(sys.argv[1])
