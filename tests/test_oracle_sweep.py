"""Pins of the ENV.md §5 offline-sweep oracle: P:257-262 (the
frequency sweep and its U-shaped EDP curves), Table 6 P:550-567 (Offline vs Online).

Every pin is a property the definition or the mathematics fixes, or a cross-check against
an independently written part of the oracle (the tuner loop's stats, §4.9):
* a tuner forced onto arm k in every window accumulates exactly S[k] (same values, same
  left-to-right order), and a tuner forced onto the per-window oracle arm k° accumulates O;
* the per-window oracle is no worse than any fixed arm (monotone rounding of sums);
* chunked sweeps equal one sweep; prototype buckets partition the windows;
* single-prototype traces put the Offline optimum inside the paper's bands with the
  compute-heavy ≥ efficiency ordering.
"""
import numpy as np
import pytest

from agft_inputs import named_config, tuner_params


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def _cfg(**kw):
    c = named_config("C2")
    c.update(kw)
    return c


def test_fixed_arm_tuner_accumulates_the_sweep_row(orc):
    """§5: a tuner that chose arm k in every window has sum_edp = S[r][k].EDP bit for bit."""
    c = _cfg(prune_enable=0, T=600)
    acc, best = orc.sweep(c, 3, 0, 600, best=True)
    for k in (0, 17, 73, 106):
        st, _, _ = orc.run_tuner(c, orc.make_tuner(3), T=600, follow=np.full(600, k, np.uint8))
        assert st["follow_violations"] >= 0
        assert st["sum_energy"] == acc["S"][k, 0]
        assert st["sum_tpot"] == acc["S"][k, 1]
        assert st["sum_edp"] == acc["S"][k, 2]
    # following the per-window oracle arm reproduces O
    st, _, _ = orc.run_tuner(c, orc.make_tuner(3), T=600, follow=best)
    assert st["sum_edp"] == acc["O"][0] and st["sum_energy"] == acc["O"][1]


def test_window_oracle_dominates_every_fixed_arm(orc):
    """Σ_t min_k EDP ≤ Σ_t EDP_k for every k (termwise ≤, rounding is monotone)."""
    for name, r in (("C2", 0), ("C4", 1), ("C4", 200)):
        c = named_config(name)
        acc, best = orc.sweep(c, r, 0, 1500, best=True)
        assert np.all(acc["O"][0] <= acc["S"][:, 2])
        k_off = orc.offline_arm(acc["S"][:, 2])
        assert acc["S"][k_off, 2] == acc["S"][:, 2].min()
        assert np.all(acc["S"][:k_off, 2] > acc["S"][k_off, 2])          # smallest minimiser
        # per-window oracle arms really minimise EDP (spot check through ENV-R)
        rows = orc.trace_rows(c, r, 0, 20)
        for t in range(20):
            edp = [orc.env_response(c, rows[t], F)[3] for F in
                   range(c["f_min_mhz"], c["f_min_mhz"] + c["n_arms"] * c["f_step_mhz"], c["f_step_mhz"])]
            assert best[t] == int(np.argmin(edp))


def test_chunked_sweep_equals_one_sweep_and_buckets_partition(orc):
    c = named_config("C4")
    one, b1 = orc.sweep(c, 129, 0, 2000, best=True)
    acc = orc.new_sweep(c)
    parts = []
    for t0, n in ((0, 1), (1, 750), (751, 500), (1251, 749)):
        acc, b = orc.sweep(c, 129, t0, n, acc, best=True)
        parts.append(b)
    for key in ("S", "SP", "NP", "O"):
        assert np.array_equal(one[key], acc[key]), key
    assert np.array_equal(np.concatenate(parts), b1)
    assert int(one["NP"].sum()) == 2000
    # the bucket of window t is its segment's prototype
    counts = np.zeros(5, np.int64)
    for t in range(0, 2000, 50):
        counts[orc.prototype(c, 129, t)] += 1
    assert set(np.nonzero(counts)[0]) <= set(np.nonzero(one["NP"])[0])
    # per-prototype sums add up to the arm totals (different association: rounding only)
    np.testing.assert_allclose(one["SP"].sum(axis=0), one["S"][:, 2], rtol=1e-12)


def test_offline_optimum_per_prototype_in_paper_bands(orc):
    """P:259-262 / Table 6: compute-heavy workloads (Long Context, High Concurrency) have
    higher EDP-optimal frequencies than the efficiency ones; all interior, 1100–1500 MHz."""
    f_off = []
    for p in range(5):
        w = [0] * 5
        w[p] = 256
        c = _cfg(weight=w)
        acc, _ = orc.sweep(c, 7, 0, 1500)
        assert acc["NP"][p] == 1500
        k = orc.offline_arm(acc["SP"][p])
        assert k == orc.offline_arm(acc["S"][:, 2])
        assert 0 < k < c["n_arms"] - 1
        f_off.append(c["f_min_mhz"] + k * c["f_step_mhz"])
    normal, longctx, longgen, highconc, hithit = f_off
    assert longctx >= normal and highconc >= normal and longctx >= hithit and highconc >= longgen
    assert all(1100 <= f <= 1500 for f in f_off), f_off


def test_regret_against_window_oracle_is_nonnegative(orc):
    """No policy beats the per-window oracle: sum_edp(i) ≥ O[r].EDP for free-running tuners."""
    c = named_config("C4")
    T = 3000
    ids = [0, 5, 15, 100, 255, 256 * 130 + 7]
    p = tuner_params(c, ids)
    stats = orc.run_batch(c, p, T, threads=4)
    for i, st in zip(ids, stats):
        acc, _ = orc.sweep(c, int(p["trace_id"][ids.index(i)]), 0, T)
        assert st["sum_edp"] >= acc["O"][0]
