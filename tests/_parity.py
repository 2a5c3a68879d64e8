"""Shared helpers of the GPU-vs-oracle parity tests (tests/ only)."""
from __future__ import annotations

import numpy as np

import oracle

EXACT_STATS = ("steps", "last_arm", "n_active", "n_pruned_extreme", "n_pruned_hist", "n_pruned_cascade",
               "sum_active", "sum_energy", "sum_tpot", "sum_ttft", "sum_edp", "sum_reward",
               "base_energy", "base_edp", "exploit_steps", "ph_alarms", "first_exploit_t", "phase",
               "n_refine", "last_anchor")
REL_TOL = 1e-9   # north_star: A⁻¹ entries and scores to 1e-9 relative (fp64)


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
            err = np.max(np.abs(gv[k] - ov[k])) / scale
            if err > REL_TOL:
                errs.append(f"{f}[{k}] rel err {err:.3e}")
                break
    return errs


def compare_tuner(cfg: dict, params: dict, i: int, gstats_row, garms: dict | None, T: int,
                  traj: np.ndarray | None = None, trace_base: int = 0) -> tuple[list[str], dict]:
    """Free-running comparison; if trajectories differ and the GPU recorded its choices,
    re-run the oracle in follow-GPU mode (ENV.md §4.5) and compare under that trajectory."""
    tu = oracle_tuner(params, i, trace_base)
    ost, oarms, _ = oracle.run_tuner(cfg, tu, T=T)
    info = {"mode": "free", "near_gpu": int(gstats_row["near_tie_steps"]), "near_orc": ost["near_tie_steps"]}
    if int(gstats_row["traj_hash"]) != ost["traj_hash"]:
        if traj is None:
            return [f"tuner {i}: trajectory hash differs and no record to follow"], info
        ost, oarms, _ = oracle.run_tuner(cfg, tu, T=T, follow=traj)
        info["mode"] = "follow"
        info["violations"] = ost["follow_violations"]
        info["max_viol_rel"] = ost["max_viol_rel"]
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
    if garms is not None:
        errs += [f"tuner {i}: {e}" for e in compare_arms(garms, oarms, cfg["n_arms"])]
    return errs, info
