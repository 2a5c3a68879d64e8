"""Block-scheduling timeline of one C4 day (agft_timeline, include/agft.h): every warp of every
replay-class launch records (launch, class, SM, start, end).  Prints, per group of launches
(a sub-chunk = the class launches between two classifications), the span, the per-class warp counts
and durations and the SM-slot utilisation, so that the gap between the per-class latency ceilings
and the concurrent day can be attributed to scheduling (tails, waves) or to the kernels.

    python tools/timeline.py [--config C4] [--chunk 4500] [--out gpurun_out/timeline.npz]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CLS = ("wide", "seg_g16", "seg_g8", "seg_g4", "solo", "seg_g32")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--T", type=int, default=None)
    ap.add_argument("--chunk", type=int, default=4500)
    ap.add_argument("--cap", type=int, default=12_000_000)
    ap.add_argument("--out", default="gpurun_out/timeline.npz")
    ap.add_argument("--json", default="gpurun_out/timeline_summary.json")
    args = ap.parse_args()

    import numpy as np
    import torch
    from paper_2508_01744_b200 import build as _build, _abi
    _abi.LIB_PATH = _build.build_variant("timeline", ["AGFT_TIMELINE=1"])   # before the first lib() call
    import paper_2508_01744_b200 as pkg
    from paper_2508_01744_b200 import TunerBatch
    from agft_inputs import named_config, tuner_params

    cfg = named_config(args.config)
    if args.T:
        cfg["T"] = args.T
    T = cfg["T"]
    params = tuner_params(cfg)
    torch.cuda.set_device(0)
    tb = TunerBatch(cfg, params, device="cuda:0")
    chunk = min(args.chunk, T)
    records = tb.new_records(chunk)
    buf = torch.zeros(1 + 3 * args.cap, dtype=torch.int64, device="cuda:0")

    def day(tl: bool):
        tb.reset()
        if tl:
            pkg.agft_timeline(tb.h, buf, args.cap)
        t = 0
        evs = []
        while t < T:
            m = min(chunk, T - t)
            pkg.agft_trace_generate(tb.h, t, m, records, None)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tb.replay(records, t, m)
            e1.record()
            evs.append((t, m, e0, e1))
            t += m
        torch.cuda.synchronize()
        if tl:
            pkg.agft_timeline(tb.h, None)
        return [(t, m, a.elapsed_time(b)) for t, m, a, b in evs]

    day(False)                                   # warm-up
    plain = day(False)
    chunks = day(True)
    n_rec = int(buf[0].item())
    assert n_rec <= args.cap, (n_rec, args.cap)
    r = buf[1:1 + 3 * n_rec].view(n_rec, 3).cpu().numpy()
    w0 = r[:, 0].astype(np.uint64)
    seq = (w0 >> np.uint64(32)).astype(np.int64)
    cls = ((w0 >> np.uint64(16)) & np.uint64(0xffff)).astype(np.int64)
    sm = (w0 & np.uint64(0xffff)).astype(np.int64)
    t0 = r[:, 1].astype(np.int64)
    t1 = r[:, 2].astype(np.int64)
    # warps past the class count exit at once (the grid covers all N tuners): drop them
    real = (t1 - t0) > 50_000
    seq, cls, sm, t0, t1 = seq[real], cls[real], sm[real], t0[real], t1[real]
    base = t0.min()
    t0 = t0 - base
    t1 = t1 - base
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    np.savez_compressed(args.out, seq=seq, cls=cls, sm=sm, t0=t0, t1=t1)

    # group launches into sub-chunks: launches of one sub-chunk are consecutive sequence numbers
    # 6k..6k+5 (one per class, in class order, every sub-chunk launches all six)
    grp = seq // 6
    n_sm = int(sm.max()) + 1
    out = {"config": args.config, "T": T, "chunk": chunk, "records": n_rec, "n_sm": n_sm,
           "day_ms_plain": sum(c[2] for c in plain), "day_ms_timeline": sum(c[2] for c in chunks),
           "subchunks": []}
    tot_busy = 0.0
    tot_span = 0.0
    for g in np.unique(grp):
        m = grp == g
        s0, s1 = t0[m].min(), t1[m].max()
        span = (s1 - s0) / 1e6
        row = {"group": int(g), "span_ms": round(span, 3), "classes": {}}
        busy = 0.0
        for c in range(6):
            mc = m & (cls == c)
            if not mc.any():
                continue
            d = (t1[mc] - t0[mc]) / 1e6
            busy += d.sum()
            row["classes"][CLS[c]] = {"warps": int(mc.sum()), "dur_ms_mean": round(float(d.mean()), 3),
                                      "dur_ms_max": round(float(d.max()), 3),
                                      "start_ms_max": round(float((t0[mc].max() - s0) / 1e6), 3),
                                      "end_ms_max": round(float((t1[mc].max() - s0) / 1e6), 3)}
        row["warp_ms"] = round(busy, 2)
        # warp slots in use over the span vs 8 per SM (the register-file limit of every class)
        row["slot_util_8_per_sm"] = round(busy / (span * n_sm * 8), 3)
        tot_busy += busy
        tot_span += span
        out["subchunks"].append(row)
    out["slot_util_day"] = round(tot_busy / (tot_span * n_sm * 8), 3)
    # occupancy over time: warps resident per SM, sampled every 0.1 ms over the whole day
    grid = np.arange(0, t1.max(), 100_000)
    ev_t = np.concatenate([t0, t1])
    ev_d = np.concatenate([np.ones_like(t0), -np.ones_like(t1)])
    o = np.argsort(ev_t, kind="stable")
    cum = np.cumsum(ev_d[o])
    idx = np.searchsorted(ev_t[o], grid, side="right") - 1
    res = np.where(idx >= 0, cum[np.clip(idx, 0, None)], 0) / n_sm
    hist, edges = np.histogram(res, bins=[0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 100])
    out["resident_warps_per_sm_hist"] = {f"{int(edges[i])}-{int(edges[i + 1])}": round(float(h) / len(res), 4)
                                         for i, h in enumerate(hist)}
    with open(args.json, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "subchunks"}))
    for row in out["subchunks"]:
        print(json.dumps(row))


if __name__ == "__main__":
    main()
