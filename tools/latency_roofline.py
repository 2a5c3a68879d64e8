"""Latency roofline per replay class.

The replay is a serial chain per tuner (Eq. 1 → argmax → ENV-R → reward → Sherman–Morrison →
Welford → pruning, PAPER §4.2–4.3), so a class kernel is bounded by
    resident tuners per GPU ÷ chain latency per window
(no throughput pipe is near saturation: ncu shows FP64 ≤ 26%, issue ≤ 40%).  For each class this
measures, on the library itself:
  * the chain latency: one warp's worth of tuners of that class alone on the GPU for n windows
    (µs and SM cycles per window at the sampled clock);
  * the residency: resident tuners per SM from agft_occupancy (CUDA occupancy calculator) × 148;
  * the throughput with exactly one full wave of that class;
and reports the ceiling, the full-wave rate and its fraction of the ceiling (what SM contention
costs).  Classes are pinned by the grid size with pruning configured never to fire (extreme
threshold −1e300, k_h = 1e300: the pruning statistics still run, nothing is removed), so K_act = K
for the whole run: K = 1 SOLO, 8 SEG G=4, 16 SEG G=8, 32 SEG G=16, 64 SEG G=32, 107 WIDE.

  python tools/latency_roofline.py [--T 4096] [--out profiles/r02_latency_roofline.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CLASSES = [("solo", 4, 1, 32), ("seg_g4", 3, 8, 8), ("seg_g8", 2, 16, 4), ("seg_g16", 1, 32, 2),
           ("seg_g32", 5, 64, 1), ("wide", 0, 107, 1)]       # name, agft_profile slot, K, tuners per warp
N_SM = 148


def sm_max_mhz():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["sm_max_mhz"])
    except (OSError, ValueError, KeyError):
        return 1965.0


def run_class(K, n, T, reps=3):
    import torch
    from agft_inputs import named_config
    from paper_2508_01744_b200 import TunerBatch
    cfg = dict(named_config("C2"), n_arms=K, n_tuners=n, n_traces=1, T=T)
    p = {"trace_id": np.zeros(n, np.uint32), "alpha0": np.ones(n), "ext_reward_threshold": np.full(n, -1e300),
         "hist_k": np.full(n, 1e300)}
    tb = TunerBatch(cfg, p, device="cuda:0")
    rec = tb.new_records(T)
    tb.generate(0, T, rec)
    stream = torch.cuda.current_stream()
    best = None
    for r in range(reps + 1):
        tb.reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tb.replay(rec, 0, T)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if r > 0:
            best = ms if best is None else min(best, ms)
    st = tb.stats()
    assert np.all(st["n_active"] == K), "class pinned"
    tb.close()
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=4096)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_latency_roofline.json"))
    args = ap.parse_args()
    import torch
    import paper_2508_01744_b200 as pkg
    from paper_2508_01744_b200 import make_config
    from agft_inputs import named_config
    torch.cuda.set_device(0)
    rows = {}
    for name, slot, K, tpw in CLASSES:
        cfg = dict(named_config("C2"), n_arms=K, n_tuners=1, n_traces=1)
        per_sm = pkg.agft_occupancy(make_config(cfg, n_tuners=1, n_traces=1), slot)
        lat_ms = run_class(K, tpw, args.T)
        n_full = per_sm * N_SM
        full_ms = run_class(K, n_full, args.T)
        clk = sm_max_mhz()                                   # the bench runs at the max clock under load
        us_per_win = lat_ms * 1e3 / args.T
        ceiling = n_full / (us_per_win * 1e-6)
        full_rate = n_full * args.T / (full_ms * 1e-3)
        rows[name] = {"K_act": K, "tuners_per_warp": tpw, "resident_tuners_per_sm": per_sm,
                      "resident_tuners_gpu": n_full,
                      "chain_latency_us_per_window": round(us_per_win, 3),
                      "chain_latency_cycles_per_window": round(us_per_win * clk, 0) if clk else None,
                      "latency_ceiling_tuner_steps_per_s": round(ceiling, 1),
                      "full_wave_tuner_steps_per_s": round(full_rate, 1),
                      "full_wave_frac_of_ceiling": round(full_rate / ceiling, 4),
                      "sm_mhz": clk}
        print(name, json.dumps(rows[name]), flush=True)
    import bench
    out = {"src_sha": bench.src_sha(), "how": "tools/latency_roofline.py: one warp of tuners alone (chain latency) and one full wave "
                  "(agft_occupancy × 148 SMs) of a class pinned by K with pruning never firing; "
                  f"T = {args.T} windows, best of 3 replays, CUDA events", "classes": rows,
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
