"""Per-kernel DRAM traffic of one bench step from an ncu --metrics csv
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum) → JSON summary."""
import collections, csv, json, sys

def main(path, out):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "second": 1.0, "s": 1.0}
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows[1:]:
        k = r[ki].split("(")[0].replace("void ", "").replace("agft::", "")
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[k][r[mi]] += v
        if r[mi] == "gpu__time_duration.sum":
            cnt[k] += 1
    rep = {}
    tot_b = tot_t = 0.0
    for k, m in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        b = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        rep[k] = {"launches": cnt[k], "time_ms": round(m["gpu__time_duration.sum"] * 1e3, 3),
                  "dram_read_bytes": m["dram__bytes_read.sum"], "dram_write_bytes": m["dram__bytes_write.sum"],
                  "dram_bytes_per_launch": round(b / max(cnt[k], 1))}
        if "replay" in k or "seg2" in k or "solo" in k or "lane" in k or "mseg" in k:
            tot_b += b
            tot_t += m["gpu__time_duration.sum"]
    rep["_replay_total"] = {"dram_bytes": tot_b, "time_ms": round(tot_t * 1e3, 3),
                            "note": "sum over the replay-class kernels of one bench step (serialised under ncu)"}
    json.dump(rep, open(out, "w"), indent=1)
    for k, v in rep.items():
        print(k, v)

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
