"""Shared helpers of the GPU-vs-oracle parity tests (tests/ only)."""
from __future__ import annotations

import numpy as np

import oracle

EXACT_STATS = ("steps", "last_arm", "n_active", "n_pruned_extreme", "n_pruned_hist", "n_pruned_cascade",
               "sum_active", "sum_energy", "sum_tpot", "sum_ttft", "sum_edp", "sum_reward",
               "base_energy", "base_edp", "exploit_steps", "ph_alarms", "first_exploit_t", "phase",
               "n_refine", "last_anchor")
REL_TOL = 1e-9   # north_star: A⁻¹ entries and scores to 1e-9 relative (fp64)
ABS_FLOOR = 1e-12  # per-entry floor, as a fraction of the arm's largest |entry| (entries that cancel to ~0)
# the recorded top-2 gap (s1 − s2)/max(m1, m2) (ENV.md §4.5): two scores each within REL_TOL of their
# magnitude move it by at most (REL_TOL·m1 + REL_TOL·m2)/max(m1, m2) ≤ 2·REL_TOL
GAP_TOL = 2 * REL_TOL
TIE_EDGE = 1e-12  # near-tie flags may differ only where the gap is within this of tie_rel


def oracle_tuner(params: dict, i: int, trace_base: int = 0):
    return oracle.make_tuner(int(params["trace_id"][i]) + trace_base, params["alpha0"][i],
                             params["ext_reward_threshold"][i], params["hist_k"][i])


def compare_arms(g: dict, o: dict, K: int) -> list[str]:
    errs = []
    for f in ("n", "active"):
        if not np.array_equal(np.asarray(g[f]).astype(np.int64), np.asarray(o[f]).astype(np.int64)):
            errs.append(f"{f} differs")
    for f in ("b", "rbar", "ebar"):          # bit-exact by ENV.md §0
        if not np.array_equal(g[f], o[f]):
            errs.append(f"{f} differs (max abs {np.max(np.abs(g[f] - o[f])):.3e})")
    for f in ("Ainv", "theta"):              # tolerance-compared (Sherman–Morrison vs Gauss–Jordan)
        gv, ov = np.asarray(g[f]), np.asarray(o[f])
        for k in range(K):
            scale = max(np.max(np.abs(ov[k])), 1e-300)
            if f == "Ainv":                  # north_star: A⁻¹ ENTRIES to 1e-9 relative (floor 1e-12 of the scale)
                tol = REL_TOL * np.abs(ov[k]) + ABS_FLOOR * scale
            else:                            # θ enters Eq. 1 only through θᵀx, x ∈ [0,1]^d: normwise per arm
                tol = np.full(ov[k].shape, REL_TOL * scale)
            bad = np.abs(gv[k] - ov[k]) > tol
            if np.any(bad):
                e = np.argmax(np.abs(gv[k] - ov[k]) - tol)
                errs.append(f"{f}[{k}] entry {np.unravel_index(e, ov[k].shape)}: gpu {gv[k].flat[e]!r} "
                            f"oracle {ov[k].flat[e]!r}")
                break
    return errs


def entry_rel_err(g: np.ndarray, o: np.ndarray) -> float:
    """max over entries of |g − o| / (|o| + 1e-3·max|o|) — the per-entry relative error reported by
    bench.py (entries 1,000× below the arm's largest are measured against that floor)."""
    g, o = np.asarray(g, np.float64), np.asarray(o, np.float64)
    scale = np.max(np.abs(o), axis=tuple(range(1, o.ndim)), keepdims=True)
    return float(np.max(np.abs(g - o) / np.maximum(np.abs(o) + 1e-3 * scale, 1e-300)))


def compare_tuner(cfg: dict, params: dict, i: int, gstats_row, garms: dict | None, T: int,
                  traj: np.ndarray | None = None, trace_base: int = 0,
                  gap: np.ndarray | None = None) -> tuple[list[str], dict]:
    """Free-running comparison; if trajectories differ and the GPU recorded its choices,
    re-run the oracle in follow-GPU mode (ENV.md §4.5) and compare under that trajectory.
    With a recorded trajectory the oracle also records its per-step top-2 gap: the GPU's
    ``gap`` (if given) must match it within GAP_TOL, and the near-tie counts must be equal
    unless some step's gap lies within TIE_EDGE of tie_rel (where the 1e-9 score tolerance can
    legitimately flip the flag)."""
    tu = oracle_tuner(params, i, trace_base)
    rec_on = traj is not None
    ost, oarms, orec = oracle.run_tuner(cfg, tu, T=T, record=rec_on)
    info = {"mode": "free", "near_gpu": int(gstats_row["near_tie_steps"]), "near_orc": ost["near_tie_steps"]}
    if int(gstats_row["traj_hash"]) != ost["traj_hash"]:
        if traj is None:
            return [f"tuner {i}: trajectory hash differs and no record to follow"], info
        ost, oarms, orec = oracle.run_tuner(cfg, tu, T=T, follow=traj, record=True)
        info["mode"] = "follow"
        info["violations"] = ost["follow_violations"]
        info["max_viol_rel"] = ost["max_viol_rel"]
        info["near_orc"] = ost["near_tie_steps"]
    errs = []
    if info.get("violations", 0):
        errs.append(f"tuner {i}: {ost['follow_violations']} GPU choices outside the near-tie set "
                    f"(worst rel gap {ost['max_viol_rel']:.3e})")
    if int(gstats_row["traj_hash"]) != ost["traj_hash"]:
        errs.append(f"tuner {i}: hash differs even in follow mode")
    for f in EXACT_STATS:
        gv = gstats_row[f]
        if gv != ost[f]:
            errs.append(f"tuner {i}: stats.{f} {gv!r} != {ost[f]!r}")
    # a6: the near-tie flag count (ENV.md §4.5)
    edge = False
    if orec is not None:
        og = orec["gap"]
        edge = bool(np.any(np.abs(og[np.isfinite(og)] - cfg["tie_rel"]) <= TIE_EDGE))
        info["gap_edge"] = edge
    if info["near_gpu"] != info["near_orc"] and not edge:
        errs.append(f"tuner {i}: near_tie_steps gpu {info['near_gpu']} != oracle {info['near_orc']}")
    if gap is not None and orec is not None:
        gg, og = np.asarray(gap[:T], np.float64), orec["gap"]
        inf_ok = np.array_equal(np.isinf(gg), np.isinf(og))
        fin = np.isfinite(og) & np.isfinite(gg)
        worst = float(np.max(np.abs(gg[fin] - og[fin]), initial=0.0))
        info["gap_max_abs_diff"] = worst
        info["gap_steps"] = int(fin.sum())
        if not inf_ok:
            errs.append(f"tuner {i}: single-arm steps (gap = inf) differ")
        if worst > GAP_TOL:
            t = int(np.argmax(np.where(fin, np.abs(gg - og), -1)))
            errs.append(f"tuner {i}: gap at step {t}: gpu {gg[t]!r} oracle {og[t]!r}")
    if garms is not None:
        errs += [f"tuner {i}: {e}" for e in compare_arms(garms, oarms, cfg["n_arms"])]
    return errs, info
