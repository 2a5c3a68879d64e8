"""Per-class DRAM traffic of one bench step from an ncu CSV launch list captured with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum, written as the
profiles/*_traffic.json that bench.py matches on (source hash, workload key).

usage: ncu_traffic.py LAUNCHES_CSV OUT_JSON WORKLOAD_KEY [DAYS]
(DAYS = replay days in the capture: `bench.py --steps 1 --warmup 0` replays the timed day and the
serialised attribution day, so 2)"""
import csv
import json
import os
import re
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (src_sha only)

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
        "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}


def slot(name: str) -> str:
    n = name.replace("(int)", "")
    if n.startswith("void solo_kernel") or n.startswith("solo_kernel"):
        return "solo"
    m = re.search(r"seg\d?_kernel<\s*\d+,\s*(\d+)", n)
    if m:
        return f"seg_g{m.group(1)}"
    m = re.search(r"replay_kernel<\s*\d+,\s*\d+,\s*(\d+)", n)
    if m:
        return {"0": "wide", "3": "refine"}.get(m.group(1), "live")
    if "class_" in n:
        return "classify"
    if "trace_kernel" in n:
        return "trace"
    return "other"


def main(path, out, key, days="2"):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(lambda: defaultdict(float))
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        per[(int(d["ID"]), d["Kernel Name"])][d["Metric Name"]] = v
    classes = defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "ncu_ms": 0.0})
    for (_, name), m in per.items():
        c = classes[slot(name)]
        c["launches"] += 1
        c["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        c["ncu_ms"] += m.get("gpu__time_duration.sum", 0.0)
    tot = sum(c["dram_bytes"] for k, c in classes.items() if k not in ("trace", "other"))
    json.dump({"src_sha": bench.src_sha(), "workload_key": key, "classes": classes, "days_in_capture": int(days),
               "total_dram_bytes": tot / int(days),
               "how": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none over every launch of one bench step (cold, serialised)"},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:5])
