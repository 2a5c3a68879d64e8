"""Attribute ncu per-instruction samples/instruction counts to kernel-body source lines.
usage: sass_attrib.py NCU_SASS_CSV NVDISASM_GI_SASS KERNEL_MANGLED_SUBSTR SRC_FILE LO HI
(NCU_SASS_CSV from `ncu -i R --page source --csv --print-source sass`; the gi file from
`nvdisasm -gi` of the same cubin)."""
import csv, re, sys, collections

def main(csvp, sassp, kern, src, lo, hi):
    lo, hi = int(lo), int(hi)
    rows = list(csv.reader(open(csvp)))
    hdr = rows[1]
    data = []
    for r in rows[2:]:
        if len(r) < len(hdr) or not r[0].startswith("0x"):
            continue
        d = dict(zip(hdr, r))
        data.append((int(r[0], 16), float(d["Warp Stall Sampling (All Samples)"] or 0), float(d["Instructions Executed"] or 0), r[1].strip()))
    base = data[0][0]
    lines = open(sassp).read().split("\n")
    start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and kern in l)
    loc = {}
    cur = "?"
    for l in lines[start + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
        if m:
            f, ln, fi, li = m.group(1), int(m.group(2)), m.group(3), m.group(4)
            if fi and fi.endswith(src) and lo <= int(li) <= hi:
                cur = f"{src}:{li}"
            elif f.endswith(src) and lo <= ln <= hi:
                cur = f"{src}:{ln}"
            else:
                cur = f"{f.split('/')[-1]}:{ln}" + (f"@{fi.split('/')[-1]}:{li}" if fi else "")
            continue
        m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
        if m:
            loc[int(m.group(1), 16)] = cur
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    for a, s, i, _ in data:
        k = loc.get(a - base, "??")
        agg[k][0] += s
        agg[k][1] += i
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    srcl = open(next(p for p in [sys.argv[7]] if p)).read().split("\n") if len(sys.argv) > 7 else None
    print(f"samples {ts:.0f} instructions {ti:.3e}")
    for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[8]) if len(sys.argv) > 8 else 60]:
        txt = ""
        if srcl and k.startswith(src + ":"):
            txt = srcl[int(k.split(":")[1]) - 1].strip()[:70]
        print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% inst {i/ti*ti:10.3e}  {k:40s} {txt}")

if __name__ == "__main__":
    main(*sys.argv[1:7])
