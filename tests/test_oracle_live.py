"""Pins of the oracle's live-controller environment: the context of
each window built from its MetricsSnapshot counters (§4.1) and a MEASURED response
(E, TPOT, TTFT) in place of ENV-R, with EDP = E × TPOT (AMB-4).  These are the inputs
agft_select / agft_observe take on the GPU (tests/test_gpu_live.py)."""
import numpy as np
import pytest

import oracle
from agft_inputs import frequencies, live_inputs, named_config, tiny_config, with_overrides


def _env_table(cfg, rows):
    """(E, TPOT, TTFT) of every arm at every window from the oracle's own ENV-R."""
    T, K = len(rows), cfg["n_arms"]
    resp = np.zeros((T, K, 3))
    for t in range(T):
        for k, f in enumerate(frequencies(cfg)):
            E, tpot, ttft, _ = oracle.env_response(cfg, rows[t], f)
            resp[t, k] = (E, tpot, ttft)
    return resp


@pytest.mark.parametrize("name,T", [("C1", 200), ("C2", 160)])
def test_live_with_the_closed_form_response_is_the_replay(name, T):
    """Feeding the live path the trace's own snapshots and the ENV-R response of every arm
    reproduces the closed-form replay step for step (ENV.md §3-§4: the environment is the only
    thing the live path swaps out).  The f_max baseline is not measurable live: base_* = 0."""
    cfg = named_config(name)
    rows = oracle.trace_rows(cfg, 0, 0, T)
    st, arms, rec = oracle.run_tuner(cfg, T=T, record=True)
    sl, al, rl = oracle.run_tuner(cfg, T=T, record=True,
                                  inject={"rows": rows, "resp": _env_table(cfg, rows)})
    assert np.array_equal(rec["arm"], rl["arm"])
    for f in ("traj_hash", "sum_energy", "sum_tpot", "sum_ttft", "sum_edp", "sum_reward",
              "n_active", "n_pruned_extreme", "n_pruned_hist", "n_pruned_cascade", "near_tie_steps"):
        assert st[f] == sl[f], f
    assert sl["base_energy"] == 0.0 and sl["base_edp"] == 0.0
    for f in ("n", "active", "b", "rbar", "ebar"):
        assert np.array_equal(arms[f], al[f]), f
    np.testing.assert_array_equal(arms["Ainv"], al["Ainv"])


def test_live_two_steps_by_hand():
    """d = 1, two arms, α0 = 1, a snapshot with waiting > 0 (x1 = 1).  Step 0: both arms are
    fresh and tie, the lowest frequency wins (AMB-5); the window is empty so r = 0 (AMB-3).
    Step 1: arm 0 has A = 2, θ = 0 → s0 = α_1·√(1/2); arm 1 is fresh → s1 = α_1 > s0, so arm 1
    runs.  With (E, TPOT) = (100 J, 0.02 s) then (50 J, 0.02 s): EDP 2.0 then 1.0, reward
    1 − 1.0/2.0 = 0.5, so b1 = 0.5, A1 = 2, θ1 = 0.25, r̄1 = 0.5, ē1 = 1.0 (P:155, P:364,
    Eqs. 3–5)."""
    cfg = tiny_config(n_arms=2, d=1, prune_enable=0)
    row = np.zeros(12, np.uint32)
    row[0] = 3                                   # waiting → x1 = 1
    rows = np.stack([row, row])
    resp = np.zeros((2, 2, 3))
    resp[0, 0] = (100.0, 0.02, 0.5)
    resp[0, 1] = (7.0, 7.0, 7.0)                 # never read: arm 0 runs at step 0
    resp[1, 1] = (50.0, 0.02, 0.25)
    resp[1, 0] = (9.0, 9.0, 9.0)                 # never read: arm 1 runs at step 1
    st, arms, rec = oracle.run_tuner(cfg, T=2, record=True, inject={"rows": rows, "resp": resp})
    assert list(rec["arm"]) == [0, 1]
    assert list(rec["edp"]) == [2.0, 1.0]
    assert list(rec["reward"]) == [0.0, 0.5]
    assert st["sum_energy"] == 150.0 and st["sum_tpot"] == 0.04 and st["sum_ttft"] == 0.75
    assert st["sum_edp"] == 3.0 and st["sum_reward"] == 0.5
    assert arms["b"][1, 0] == 0.5 and arms["theta"][1, 0] == 0.25
    assert arms["Ainv"][1, 0, 0] == 0.5 and arms["Ainv"][0, 0, 0] == 0.5
    assert arms["rbar"][1] == 0.5 and arms["ebar"][1] == 1.0 and arms["ebar"][0] == 2.0


def test_live_inputs_drive_a_bandit_to_the_cheap_arms():
    """On the seeded live inputs the tuner's mean EDP over the second half beats a uniformly
    random controller's expected EDP on the same windows (a regret sanity check)."""
    cfg = with_overrides(named_config("C2"), prune_enable=1)
    T = 1500
    rows, resp = live_inputs(cfg, 1, T, seed=7)
    st, arms, rec = oracle.run_tuner(cfg, T=T, record=True, inject={"rows": rows[0], "resp": resp[0]})
    edp_all = resp[0, :, :, 0] * resp[0, :, :, 1]
    half = slice(T // 2, T)
    assert rec["edp"][half].mean() < 0.8 * edp_all[half].mean()
    assert st["n_active"] >= 1
