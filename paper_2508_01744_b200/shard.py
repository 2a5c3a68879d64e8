"""Tuner sharding across ranks — host logic only.

Tuners never communicate, so a rank owns a contiguous block of tuner ids whose traces are
a contiguous block of trace ids: it generates its own traces (no input exchange) and the
only collective is the final all-gather of per-tuner statistics (north_star).

* ``weak``   — every rank runs the full named config; rank r's traces are offset by
  r·n_traces (a different synthetic day per rank), so total work grows with the rank count.
* ``strong`` — the named config's tuners/traces are split evenly across ranks.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Shard:
    rank: int
    world: int
    n_tuners: int          # local tuners
    n_traces: int          # local traces
    trace_base: int        # global id of local trace 0
    tuner_base: int        # global id of local tuner 0
    params: dict           # per-tuner params with LOCAL trace ids


def plan(cfg: dict, world: int, rank: int, scaling: str = "weak") -> Shard:
    from agft_inputs import tuner_params
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    N, R = cfg["n_tuners"], cfg["n_traces"]
    if scaling == "weak":
        p = tuner_params(cfg)
        return Shard(rank, world, N, R, rank * R, rank * N, p)
    if scaling != "strong":
        raise ValueError(scaling)
    if N % world or R % world:
        raise ValueError(f"{N} tuners / {R} traces do not split over {world} ranks")
    n, r = N // world, R // world
    ids = np.arange(rank * n, (rank + 1) * n)
    p = tuner_params(cfg, ids)
    tr = p["trace_id"].astype(np.int64)
    base = rank * r
    if tr.min() < base or tr.max() >= base + r:
        raise ValueError("tuner→trace layout does not align with the trace split")
    p["trace_id"] = (tr - base).astype(np.uint32)
    return Shard(rank, world, n, r, base, rank * n, p)


COUNTER_NAMES = ("tuner_steps", "flagged_tuners", "near_tie_steps", "incomplete_tuners", "pruned_extreme",
                 "pruned_hist", "pruned_cascade", "active_arm_steps", "exploit_steps", "ph_alarms", "refinements",
                 "tuners", "active_arms_end", "single_arm_tuners", "reserved14", "reserved15")


def counter_vector(st, T: int) -> list:
    """The 16 run counters SURVEY §8(e) all-reduces across ranks, from a rank's agft_tuner_stats
    array: tuner-steps, flagged (frozen) tuners, near-tie steps, invariant violations (tuners that did
    not complete all T steps), pruning counts by cause, Σ K_act, phase / refinement counters, tuners,
    active arms at the end and single-arm tuners."""
    s64 = lambda f: int(np.sum(st[f], dtype=np.int64))
    return [s64("steps"), int(np.count_nonzero(st["flags"])), s64("near_tie_steps"),
            int(np.count_nonzero(st["steps"] != T)), s64("n_pruned_extreme"), s64("n_pruned_hist"),
            s64("n_pruned_cascade"), int(np.sum(st["sum_active"], dtype=np.uint64)), s64("exploit_steps"),
            s64("ph_alarms"), s64("n_refine"), len(st), s64("n_active"), int(np.count_nonzero(st["n_active"] == 1)),
            0, 0]


def reduce_counters(vec, device=None, group=None) -> dict:
    """Sum-all-reduce a rank's 16 counters (one int64 tensor, one collective)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(vec, dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    return dict(zip(COUNTER_NAMES, (int(v) for v in t.cpu().tolist())))


def gather_stats(stats_bytes, group=None):
    """All-gather each rank's per-tuner stats (a uint8 tensor) in rank order (global tuner order)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty(world * stats_bytes.numel(), dtype=stats_bytes.dtype, device=stats_bytes.device)
    dist.all_gather_into_tensor(out, stats_bytes, group=group)
    return out


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank duration (timing rule: device time is the max over ranks)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
