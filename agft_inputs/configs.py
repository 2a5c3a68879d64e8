"""Named workload configurations C1–C5 and per-tuner sweep tables.

This module holds INPUTS only — constants and seeded parameter tables — and none
of the method's arithmetic. Both the CPU oracle (``oracle/``) and the CUDA path
(``paper_2508_01744_b200``) are driven from it; neither imports the other.

Sources: BASELINE.json ``configs``; ENV.md §2.1/§3 for
the environment constants; PAPER.md P:257 (210–1800 MHz, 15 MHz grid),
P:387-391 (pruning defaults), P:212-218 (Table 1 prototypes).
"""
from __future__ import annotations

import copy
import math

import numpy as np

BASE_SEED = 2508017440  # S0, SURVEY §8(d)

# Table 1 + the segment mix (ENV.md §2.1)
PROTOTYPES = {
    "names": ["Normal", "Long Context", "Long Generation", "High Concurrency", "High Cache Hit"],
    "ctx_lo": [256, 1024, 1, 256, 256],
    "ctx_hi": [1024, 8192, 256, 1024, 1024],
    "gen_lo": [100, 1, 350, 100, 100],
    "gen_hi": [350, 100, 350, 350, 350],
    "conc_mult": [1.0, 1.0, 1.0, 5.0, 1.0],
    "hit_rate": [0.05, 0.05, 0.05, 0.05, 0.90],
    "weight": [48, 112, 16, 40, 40],
}

DIURNAL_KNOTS = [0.55, 0.45, 0.38, 0.32, 0.30, 0.33, 0.40, 0.50, 0.62, 0.74, 0.84, 0.91,
                 0.96, 0.99, 1.00, 0.98, 0.94, 0.89, 0.83, 0.78, 0.74, 0.70, 0.65, 0.60]

PATTERN_FLUCT, PATTERN_DIURNAL, PATTERN_BURST, PATTERN_MOD3, PATTERN_ALT = 0, 1, 2, 3, 4

_BASE = {
    # grid
    "f_min_mhz": 210, "f_step_mhz": 15, "n_arms": 107, "f_max_hw_mhz": 1800,
    "d": 7,
    # policy (AMB-1, AMB-3)
    "alpha0": 1.0, "tau": 200.0, "median_window": 64, "clip_lo": -2.0, "clip_hi": 2.0,
    "tie_rel": 1e-9,
    # Page-Hinkley exploitation switch (ENV.md §4.10): off in C1–C5 (the §8(a) hot path)
    "ph_enable": 0, "ph_window": 50, "ph_delta": 0.005, "ph_lambda": 0.25,
    # mixed maturity-based refinement (ENV.md §4.11): off in C1–C5
    "rf_enable": 0, "rf_period": 25, "rf_mature": 100, "rf_min_samples": 4, "rf_half_mhz": 150,
    "rf_step_mhz": 15,
    # ENV-C closed loop (ENV.md §6): off in C1–C5; backlog cap 4·cap
    "cl_enable": 0, "cl_q_max": 256,
    # pruning
    "prune_enable": 1, "ext_round_limit": 60, "ext_min_samples": 3, "ext_reward_threshold": -1.2,
    "hist_min_round": 30, "hist_min_samples": 6, "hist_k": 1.0, "cascade_fraction": 0.5,
    # ENV-R (ENV.md §3)
    "W": 0.8, "p_idle": 75.0, "k_lin": 8.0, "k_cube": 21.0, "u_floor": 0.1, "u_max": 0.65,
    "c_p": 4.3e-5, "c_d": 0.0118, "beta": 0.67, "sigma_e": 0.03, "sigma_t": 0.05,
    # ENV-T (ENV.md §2.1)
    "lambda0": 2.9, "seg_steps": 750, "steps_per_hour": 4500, "burst_steps": 75,
    "burst_p32": 214748365, "burst_mult": 5.0, "cap": 64, "t_iter0": 0.0186, "t_iter1": 0.00019,
    "e2e0": 0.2, "tau_ref": 0.025, "kv_total": 262144, "pattern_mode": PATTERN_FLUCT,
    "ctx_lo": PROTOTYPES["ctx_lo"], "ctx_hi": PROTOTYPES["ctx_hi"],
    "gen_lo": PROTOTYPES["gen_lo"], "gen_hi": PROTOTYPES["gen_hi"],
    "conc_mult": PROTOTYPES["conc_mult"], "hit_rate": PROTOTYPES["hit_rate"],
    "weight": PROTOTYPES["weight"], "knot": DIURNAL_KNOTS,
    # normalisation bounds (AMB-14): x1..x7
    "norm_lo": [0.0] * 7,
    "norm_hi": [1.0, 20000.0, 2500.0, 600.0, 64.0, 1.0, 1.0],
    "seed": BASE_SEED,
    # batch shape
    "n_tuners": 1, "n_traces": 1, "T": 1000, "sweep": "none",
}

# 16 α0 values log-spaced 0.05–5 and 4×4 pruning settings
ALPHA_GRID = [0.05 * (100.0 ** (i / 15.0)) for i in range(16)]
TAU_E_GRID = [-0.6, -0.9, -1.2, -1.5]
K_H_GRID = [0.5, 1.0, 2.0, 4.0]


def named_config(name: str) -> dict:
    """Return the full parameter dict for C1..C5 (BASELINE.json ``configs``)."""
    c = copy.deepcopy(_BASE)
    c["name"] = name
    if name == "C1":    # 1 tuner, 8 arms, d=4, 1,000 steps, no pruning
        c.update(f_step_mhz=225, n_arms=8, d=4, T=1000, prune_enable=0,
                 weight=[256, 0, 0, 0, 0])                       # Normal load only (AMB-18)
    elif name == "C2":  # 1 tuner, full grid, d=7, 1 h fluctuating, pruning on
        c.update(T=4500)
    elif name == "C3":  # 4,096 tuners (seed sweep), 1 h
        c.update(T=4500, n_tuners=4096, n_traces=4096)
    elif name == "C4":  # 65,536 tuners: 16 α × 16 pruning settings × 256 traces, 24 h
        c.update(T=108000, n_tuners=65536, n_traces=256, pattern_mode=PATTERN_ALT, sweep="hyper256")
    elif name == "C5":  # 1,048,576 tuners, 4,096 traces, 24 h
        c.update(T=108000, n_tuners=1048576, n_traces=4096, pattern_mode=PATTERN_MOD3, sweep="hyper256")
    else:
        raise KeyError(name)
    return c


def with_overrides(cfg: dict, **kw) -> dict:
    c = copy.deepcopy(cfg)
    c.update(kw)
    return c


def tuner_params(cfg: dict, tuner_ids=None, trace_base: int = 0):
    """Per-tuner (trace_id, alpha0, ext_reward_threshold, hist_k) as numpy arrays.

    Layout: tuner id = [trace (slowest) | hyperparameter point (fastest)];
    within a point, α is fastest. ``trace_base`` offsets trace ids (a rank's shard).
    """
    n = cfg["n_tuners"]
    ids = np.arange(n, dtype=np.int64) if tuner_ids is None else np.asarray(tuner_ids, dtype=np.int64)
    if cfg["sweep"] == "hyper256":
        per = n // cfg["n_traces"]
        trace = ids // per
        h = ids % per
        alpha = np.asarray(ALPHA_GRID)[h % 16]
        pi = (h // 16) % 16
        tau_e = np.asarray(TAU_E_GRID)[pi // 4]
        k_h = np.asarray(K_H_GRID)[pi % 4]
    else:
        trace = ids % cfg["n_traces"]
        alpha = np.full(len(ids), cfg["alpha0"])
        tau_e = np.full(len(ids), cfg["ext_reward_threshold"])
        k_h = np.full(len(ids), cfg["hist_k"])
    return {
        "trace_id": (trace + trace_base).astype(np.uint32),
        "alpha0": alpha.astype(np.float64),
        "ext_reward_threshold": tau_e.astype(np.float64),
        "hist_k": k_h.astype(np.float64),
    }


def frequencies(cfg: dict):
    """Arm k ↔ f_min + k·step MHz (D5). Integer table — no method arithmetic."""
    return [cfg["f_min_mhz"] + k * cfg["f_step_mhz"] for k in range(cfg["n_arms"])]


def live_inputs(cfg: dict, n_tuners: int, T: int, seed: int = BASE_SEED):
    """Seeded inputs of the live controller API (agft_select / agft_observe).

    rows [n_tuners][T][12] uint32: MetricsSnapshot counters per window in ENV.md §2.2 word order
    (waiting, running, prefill, decode, iters, kv_used, hits, misses; words 8..11 unused) drawn
    independently per window — a live server's counters, with idle windows (15%) and queueing
    windows (30% with waiting > 0).
    resp [n_tuners][T][K][3] fp64: the (energy J, TPOT s, TTFT s) a measurement would return if
    arm k ran window t — a noisy U-shaped EDP over the grid whose minimum moves with the load,
    standing in for NVML / the serving engine.  Plain numpy draws: inputs, not the method."""
    rng = np.random.default_rng(seed)
    K = cfg["n_arms"]
    rows = np.zeros((n_tuners, T, 12), dtype=np.uint32)
    running = rng.integers(0, cfg["cap"] + 1, size=(n_tuners, T))
    idle = rng.random((n_tuners, T)) < 0.15
    running[idle] = 0
    iters = np.where(running > 0, rng.integers(20, 44, size=(n_tuners, T)), 0)
    waiting = np.where(rng.random((n_tuners, T)) < 0.30, rng.integers(1, 40, size=(n_tuners, T)), 0)
    arrivals = np.where(idle, 0, rng.integers(0, 12, size=(n_tuners, T)))
    hits = (arrivals * rng.random((n_tuners, T))).astype(np.int64)
    rows[..., 0] = waiting
    rows[..., 1] = running
    rows[..., 2] = arrivals * rng.integers(1, 4096, size=(n_tuners, T))
    rows[..., 3] = running * iters
    rows[..., 4] = iters
    rows[..., 5] = np.minimum(cfg["kv_total"], running * rng.integers(64, 4096, size=(n_tuners, T)))
    rows[..., 6] = hits
    rows[..., 7] = arrivals - hits
    f = np.asarray(frequencies(cfg), dtype=np.float64) / 1000.0            # GHz
    load = (running / max(cfg["cap"], 1)).astype(np.float64)[..., None]     # [N][T][1]
    f_opt = 0.9 + 0.6 * load                                               # EDP minimum moves with load
    power = 70.0 + 25.0 * f[None, None, :] ** 3 * (0.2 + load)
    tpot = 0.012 * (1.0 + 0.8 * (f_opt / f[None, None, :] - 1.0) ** 2 + 0.5 * (f_opt > f[None, None, :]))
    noise = rng.random((n_tuners, T, K, 3))
    resp = np.empty((n_tuners, T, K, 3), dtype=np.float64)
    resp[..., 0] = power * cfg["W"] * (0.97 + 0.06 * noise[..., 0])
    resp[..., 1] = tpot * (0.95 + 0.10 * noise[..., 1])
    resp[..., 2] = 0.05 + 0.2 * noise[..., 2] / f[None, None, :]
    return rows, resp


def tiny_config(**kw) -> dict:
    """A small config for oracle-only unit tests."""
    c = named_config("C2")
    c.update(kw)
    return c


assert abs(ALPHA_GRID[0] - 0.05) < 1e-15 and abs(ALPHA_GRID[-1] - 5.0) < 1e-12
assert math.isclose(sum(PROTOTYPES["weight"]), 256)
