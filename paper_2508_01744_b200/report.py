"""Reporting over the stats API: the paper's Tables 2–5 as host reductions.

The paper reports, for one serving run, the mean of each per-window metric under AGFT against
the default-clock baseline ("Normal", the f_max clock) before and after convergence (Tables 2–3,
P:440-455), and the coefficient of variation (CV = std / mean over the windows of the
run) of the full framework against two ablations: a coarse grid ("No-grain", Table 4)
and pruning disabled ("No pruning", Table 5).

Nothing here computes a step of the method.  ``windowed`` drives the CUDA replay
(``agft_trace_generate`` + ``agft_replay``) in buckets of windows and differences the cumulative
``agft_tuner_stats`` sums that ``agft_stats`` returns after each bucket; the tables are numpy
means and CVs over those series.  Readings: the baseline TPOT of a window is
base_edp / base_energy (EDP = E × TPOT); CVs are population CVs over windows, per tuner, then
averaged over tuners; the convergence round is the tuner's first Exploitation round (ENV.md
§4.10) when the phase switch is on, else the caller's split (the paper's run converged
at round 231); the No-grain grid is 120 MHz, the paper does not state it.
ENV-R has no end-to-end latency, so the paper's E2E row is not reported.
"""
from __future__ import annotations

import argparse
import json

import numpy as np

SERIES = ("energy", "tpot", "ttft", "edp", "reward", "base_energy", "base_edp")
_CUM = {"energy": "sum_energy", "tpot": "sum_tpot", "ttft": "sum_ttft", "edp": "sum_edp",
        "reward": "sum_reward", "base_energy": "base_energy", "base_edp": "base_edp"}
NO_GRAIN_STEP_MHZ = 120


def windowed(tb, T: int, bucket: int = 1) -> dict:
    """Replay windows [tb.t, T) of every tuner in buckets of ``bucket`` windows; return per-bucket
    sums {name: [n_buckets][N]} for SERIES plus "steps" [n_buckets][N] and "t0" [n_buckets], by
    differencing the cumulative stats after each bucket (host reduction over agft_stats)."""
    if bucket < 1:
        raise ValueError("bucket must be ≥ 1")
    t = tb.t
    prev = tb.stats()
    out = {k: [] for k in SERIES}
    out["steps"], out["t0"] = [], []
    rec = raw = None
    closed = bool(getattr(tb, "closed", False))
    while t < T:
        m = min(bucket, T - t)
        if rec is None or rec.shape[1] != m:
            rec = tb.new_records(m)
        if closed:                                    # ENV-C needs the raw rows (ENV.md §6)
            rec, raw = tb.generate(t, m, rec, raw=True)
        else:
            tb.generate(t, m, rec)
        tb.replay(rec, t, m, raw=raw) if closed else tb.replay(rec, t, m)
        cur = tb.stats()
        for k in SERIES:
            out[k].append(cur[_CUM[k]] - prev[_CUM[k]])
        out["steps"].append(cur["steps"].astype(np.int64) - prev["steps"].astype(np.int64))
        out["t0"].append(t)
        prev = cur
        t += m
    res = {k: np.asarray(v) for k, v in out.items()}
    res["final"] = prev
    return res


def per_window(series: dict) -> dict:
    """Per-window means of each bucket {metric: [n_buckets][N]} with the baseline TPOT."""
    n = np.maximum(series["steps"], 1).astype(np.float64)
    m = {k: series[k] / n for k in SERIES}
    with np.errstate(invalid="ignore", divide="ignore"):
        m["base_tpot"] = np.where(series["base_energy"] > 0, series["base_edp"] / series["base_energy"], np.nan)
    return m


def mean_cv(x: np.ndarray) -> tuple[float, float]:
    """Mean over tuners of the per-tuner mean and population CV of a [windows][N] series."""
    x = np.asarray(x, dtype=np.float64)
    mu = x.mean(axis=0)
    sd = x.std(axis=0)
    with np.errstate(invalid="ignore", divide="ignore"):
        cv = np.where(mu != 0, sd / np.abs(mu), np.nan)
    return float(mu.mean()), float(np.nanmean(cv)) if np.any(np.isfinite(cv)) else float("nan")


def pct(a: float, b: float) -> float:
    """(a − b)/b in percent."""
    return float("nan") if b == 0 else 100.0 * (a - b) / b


def phase_tables(series: dict, split: int | np.ndarray) -> dict:
    """Tables 2–3: AGFT vs Normal (f_max) means before and after the convergence round.
    ``split`` is one round for every tuner or an [N] array (e.g. stats.first_exploit_t + 1)."""
    w = per_window(series)
    t0 = np.asarray(series["t0"])[:, None]
    split = np.broadcast_to(np.asarray(split, dtype=np.int64), w["energy"].shape[1:])
    out = {}
    for name, sel in (("pre", t0 < split[None, :]), ("post", t0 >= split[None, :])):
        rows = {}
        for metric, base in (("energy", "base_energy"), ("edp", "base_edp"), ("tpot", "base_tpot"),
                             ("ttft", None)):
            a = np.where(sel, w[metric], np.nan)
            am = float(np.nanmean(a)) if np.any(sel) else float("nan")
            if base is None:
                rows[metric] = {"agft": am, "normal": None, "diff_pct": None}
                continue
            b = np.where(sel, w[base], np.nan)
            bm = float(np.nanmean(b)) if np.any(sel) else float("nan")
            rows[metric] = {"agft": am, "normal": bm, "diff_pct": pct(am, bm)}
        rows["windows"] = int(sel.sum())
        out[name] = rows
    return out


def ablation_configs(cfg: dict) -> dict:
    """The full framework and the two ablations of Tables 4–5 on the same traces."""
    f_min, f_top = cfg["f_min_mhz"], cfg["f_min_mhz"] + (cfg["n_arms"] - 1) * cfg["f_step_mhz"]
    coarse = dict(cfg, f_step_mhz=NO_GRAIN_STEP_MHZ, n_arms=(f_top - f_min) // NO_GRAIN_STEP_MHZ + 1)
    return {"full": dict(cfg), "no_grain": coarse, "no_pruning": dict(cfg, prune_enable=0)}


def cv_table(per_variant: dict) -> dict:
    """Tables 4–5: mean and CV of each metric per variant, and each ablation's difference to the
    full framework ((ablation − full)/full, in percent)."""
    res = {}
    for v, series in per_variant.items():
        w = per_window(series)
        res[v] = {m: dict(zip(("mean", "cv"), mean_cv(w[m]))) for m in ("energy", "edp", "tpot", "ttft")}
    full = res["full"]
    for v in res:
        if v == "full":
            continue
        for m, d in res[v].items():
            d["mean_diff_pct"] = pct(d["mean"], full[m]["mean"])
            d["cv_diff_pct"] = pct(d["cv"], full[m]["cv"])
    return res


def run_ablation(cfg: dict, params: dict, T: int, bucket: int = 1, device="cuda") -> dict:
    """Run the three variants through the CUDA path and reduce them (Tables 4–5)."""
    from . import TunerBatch
    per = {}
    for v, c in ablation_configs(cfg).items():
        tb = TunerBatch(c, params, device=device)
        per[v] = windowed(tb, T, bucket)
        tb.close()
    return {"tables": cv_table(per), "series": per}


def main(argv=None):
    from agft_inputs import named_config, tuner_params
    ap = argparse.ArgumentParser(description="Tables 2–5 of the paper from the CUDA replay")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--T", type=int, default=1500, help="windows (0.8 s each)")
    ap.add_argument("--tuners", type=int, default=16)
    ap.add_argument("--bucket", type=int, default=1, help="windows per stats snapshot (1 = per-window CVs)")
    ap.add_argument("--split", type=int, default=231, help="convergence round when the phase switch is off")
    ap.add_argument("--phase", action="store_true", help="enable the Page-Hinkley switch (split = first_exploit_t)")
    ap.add_argument("--closed", action="store_true", help="ENV-C closed-loop environment (ENV.md §6)")
    args = ap.parse_args(argv)
    cfg = dict(named_config(args.config), n_tuners=args.tuners, n_traces=args.tuners, sweep="none")
    if args.phase:
        cfg["ph_enable"] = 1
    if args.closed:
        cfg["cl_enable"] = 1
    params = tuner_params(cfg)
    ab = run_ablation(cfg, params, args.T, args.bucket)
    full = ab["series"]["full"]
    split = args.split
    if args.phase:
        fe = full["final"]["first_exploit_t"].astype(np.int64)
        split = np.where(fe == 0xFFFFFFFF, args.T, fe + 1)
    print(json.dumps({"config": args.config, "T": args.T, "tuners": args.tuners, "bucket": args.bucket,
                      "tables_2_3": phase_tables(full, split), "tables_4_5": ab["tables"]}, indent=1))


if __name__ == "__main__":
    main()
