"""Pins of the oracle's closed-loop environment ENV-C (ENV.md §6; SURVEY §8(f) NEXT row 3;
P:129-131: requests a window cannot serve keep waiting into the next one)."""
import numpy as np
import pytest

import oracle
from agft_inputs import named_config, with_overrides


def _row(waiting=0, running=10, prefill=0, decode=1000, iters=100, kv=0, hits=5, misses=5):
    return np.array([waiting, running, prefill, decode, iters, kv, hits, misses, 0, 0, 0, 0], np.uint32)


def _cfg(**kw):
    # dec(1800 MHz) = c_d / (β + (1−β)·1) = c_d exactly; prefill 0 so t_pre = 0
    return with_overrides(named_config("C2"), cl_enable=1, c_d=0.02, **kw)


def test_backlog_by_hand():
    """100 iterations × 0.02 s at f_max = 2.0 s of work in a 0.8-s window: u = 2.5, so of
    D = 10 arrivals floor(10 / 2.5) = 4 are served and 6 wait; with those 6 carried in,
    D = 16, 6 served, 10 wait; q_max caps the carry."""
    c = _cfg()
    assert oracle.closed_next(c, _row(), 0, 1800) == 6
    assert oracle.closed_next(c, _row(), 6, 1800) == 10
    assert oracle.closed_next(_cfg(cl_q_max=8), _row(), 6, 1800) == 8
    light = _row(iters=30)                       # 0.6 s of work: u = 0.75 ≤ 1, everything served
    assert oracle.closed_next(c, light, 0, 1800) == 0 and oracle.closed_next(c, light, 40, 1800) == 0


def test_backlog_never_falls_with_the_clock():
    """A lower clock means more work per window (ENV-R: dec and pre grow as f falls), so the
    carried backlog is non-increasing in F, and positive whenever u > 1."""
    c = _cfg()
    for q in (0, 5, 30):
        qs = [oracle.closed_next(c, _row(iters=40, prefill=300), q, 210 + 15 * k) for k in range(107)]
        assert all(a >= b for a, b in zip(qs, qs[1:])), qs
        assert qs[0] > 0


def test_zero_cap_is_the_open_loop():
    """q_max = 0 keeps every backlog at 0: ENV-C reduces to §2–§3 bit for bit (baseline too)."""
    base = named_config("C2")
    T = 400
    so, ao, ro = oracle.run_tuner(base, T=T, record=True)
    sc, ac, rc = oracle.run_tuner(with_overrides(base, cl_enable=1, cl_q_max=0), T=T, record=True)
    assert np.array_equal(ro["arm"], rc["arm"]) and not rc["backlog"].any()
    for f in ("traj_hash", "sum_energy", "sum_tpot", "sum_ttft", "sum_edp", "sum_reward", "base_energy",
              "base_edp"):
        assert so[f] == sc[f], f


def test_overloaded_single_arm_server_queues():
    """One arm at 210 MHz under burst load: the backlog builds (and the next window's x1 = 1
    whenever it does), and waiting requests only lengthen TTFT, so Σ TTFT and the baseline's
    sums are ≥ the open loop's on the same trace."""
    base = with_overrides(named_config("C2"), n_arms=1, pattern_mode=2, T=2000, prune_enable=0)
    so, _, ro = oracle.run_tuner(base, T=2000, record=True)
    sc, _, rc = oracle.run_tuner(with_overrides(base, cl_enable=1), T=2000, record=True)
    q = rc["backlog"]
    assert q.max() > 0 and q.max() <= 256
    carried = np.nonzero(q[:-1] > 0)[0] + 1
    assert np.all(rc["x"][carried, 0] == 1.0)
    assert sc["sum_ttft"] > so["sum_ttft"]
    assert sc["base_energy"] >= so["base_energy"] and sc["base_edp"] >= so["base_edp"]
    assert np.all(rc["ttft"] >= ro["ttft"])
