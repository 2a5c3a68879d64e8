"""Pins of the oracle's mixed maturity-based refinement (ENV.md §4.11):
SPEC's worked examples for the anchor and the refined window, and run-level invariants."""
import numpy as np

from agft_inputs import frequencies, named_config

NEVER = 0xFFFFFFFF


def _k(f):
    return (f - 210) // 15


def test_refine_window_spec_examples(orc):
    """S:331-333 on the grid (210, 1800, 15): anchor 1230 → 21 arms 1080…1380; anchor 300 →
    17 arms 210…450 (lower clamp); anchor 1800 → 11 arms 1650…1800 (upper clamp)."""
    c = named_config("C2")
    f = np.array(frequencies(c))
    for anchor, n, lo, hi in ((1230, 21, 1080, 1380), (300, 17, 210, 450), (1800, 11, 1650, 1800)):
        m = orc.refine_window(c, _k(anchor))
        assert m.sum() == n and f[m == 1].min() == lo and f[m == 1].max() == hi, anchor
        assert np.all(np.diff(f[m == 1]) == 15)


def test_refine_window_excludes_extreme_and_respects_step(orc):
    c = named_config("C2")
    ex = np.zeros(107, np.uint8)
    ex[_k(1095)] = ex[_k(1380)] = 1
    m = orc.refine_window(c, _k(1230), ex)
    assert m.sum() == 19 and m[_k(1095)] == 0 and m[_k(1380)] == 0
    # a 30-MHz refine step keeps every other grid frequency: 1080, 1110, …, 1380
    m30 = orc.refine_window(dict(c, rf_step_mhz=30), _k(1230))
    assert m30.sum() == 11
    # C1's 225-MHz grid has no other frequency within ±150 MHz: the window is the anchor alone
    c1 = named_config("C1")
    assert orc.refine_window(c1, 3).tolist() == [0, 0, 0, 1, 0, 0, 0, 0]


def test_statistical_anchor_spec_examples(orc):
    """{1230: (n=4, EDP 2.4), 1500: (n=6, EDP 3.1)} → 1230; all n < 4 → none;
    two arms tied at 2.4 → the lower frequency; an extreme-pruned arm is never the anchor."""
    c = named_config("C2")
    n = np.zeros(107, np.uint32)
    e = np.zeros(107)
    n[_k(1230)], e[_k(1230)] = 4, 2.4
    n[_k(1500)], e[_k(1500)] = 6, 3.1
    assert orc.stat_anchor(c, n, e) == _k(1230)
    n3 = np.minimum(n, 3)
    assert orc.stat_anchor(c, n3, e) is None
    n[_k(1200)], e[_k(1200)] = 5, 2.4
    assert orc.stat_anchor(c, n, e) == _k(1200)
    ex = np.zeros(107, np.uint8)
    ex[_k(1200)] = 1
    assert orc.stat_anchor(c, n, e, ex) == _k(1230)


def test_refinement_invariants_on_a_run(orc):
    """right after every refinement |active| ≤ 21 and every active arm lies within
    ±150 MHz of the anchor; the chosen arm is always active; refinements fire every 25 rounds
    once an anchor exists (statistical before t = 100, predictive after)."""
    c = dict(named_config("C2"), rf_enable=1, T=1500)
    st, _, rec = orc.run_tuner(c, orc.make_tuner(0, 1.0), T=1500, record=True)
    f = np.array(frequencies(c))
    assert st["n_refine"] >= 1500 // 25 - 4 and st["last_anchor"] != NEVER
    for t in range(24, 1500, 25):
        m = rec["active_mask"][t]
        act = np.array([(m[k // 32] >> (k % 32)) & 1 for k in range(107)], bool)
        if act.sum() <= 21:
            span = f[act]
            assert span.max() - span.min() <= 300
    for t in range(1, 1500):
        m = rec["active_mask"][t - 1]
        k = int(rec["arm"][t])
        assert (m[k // 32] >> (k % 32)) & 1


def test_extreme_pruned_arms_never_return(orc):
    """S:336 (permanence): with only extreme pruning active (historical never reached,
    no cascade region), every arm removed before the first refinement is Extreme-pruned and
    must stay out of every refined window."""
    c = dict(named_config("C2"), rf_enable=1, T=600, hist_min_round=10**9, cascade_fraction=0.05,
             ext_round_limit=24, ext_min_samples=1)
    st, _, rec = orc.run_tuner(c, orc.make_tuner(1, 2.0, ext_reward_threshold=-0.2), T=600, record=True)
    m0 = rec["active_mask"][23]
    removed = [k for k in range(107) if not (m0[k // 32] >> (k % 32)) & 1]
    assert st["n_pruned_extreme"] == len(removed) and len(removed) > 0
    for t in range(24, 600):
        m = rec["active_mask"][t]
        assert all(not (m[k // 32] >> (k % 32)) & 1 for k in removed), t


def test_period_beyond_T_equals_disabled(orc):
    base = dict(named_config("C2"), T=500)
    a, _, _ = orc.run_tuner(base, orc.make_tuner(3, 0.5), T=500)
    b, _, _ = orc.run_tuner(dict(base, rf_enable=1, rf_period=10**6), orc.make_tuner(3, 0.5), T=500)
    assert b["n_refine"] == 0 and b["last_anchor"] == NEVER
    for k in ("traj_hash", "sum_edp", "n_active", "n_pruned_hist"):
        assert a[k] == b[k], k
