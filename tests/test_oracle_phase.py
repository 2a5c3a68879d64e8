"""Pins of the oracle's exploitation phase (ENV.md §4.10; Eq. 2; S:187-195,
S:216-217): the Page-Hinkley detector against SPEC's worked examples and hand-computed
streams, and the Exploitation phase against Eq. 2 (greedy = the α = 0 special case)."""
import numpy as np

from agft_inputs import named_config

NEVER = 0xFFFFFFFF


def _cfg(**kw):
    c = named_config("C2")
    c.update(ph_enable=1, ph_window=50, ph_delta=0.005, ph_lambda=0.25, prune_enable=0,
             n_arms=4, d=3, T=200)
    c.update(kw)
    return c


def _stream(orc, cfg, rewards, seed=3):
    """Run the bandit on a synthetic context stream whose reward (for every arm) is rewards[t]."""
    T = len(rewards)
    rng = np.random.default_rng(seed)
    x = rng.random((T, cfg["d"]))
    r = np.repeat(np.asarray(rewards, float)[:, None], cfg["n_arms"], axis=1)
    st, _, _ = orc.run_tuner(cfg, T=T, inject={"x": x, "reward": r})
    return st


def test_constant_stream_is_stable_at_round_W(orc):
    """a constant reward stream of length W → stable at round W (0-based t = W − 1):
    every observation adds (r − mean − δ) = −δ, so cum − min stays 0 and never alarms."""
    for W in (1, 7, 50):
        st = _stream(orc, _cfg(ph_window=W), [0.3] * 120)
        assert st["first_exploit_t"] == W - 1 and st["ph_alarms"] == 0 and st["phase"] == 1
        assert st["exploit_steps"] == 120 - W           # greedy from step W on


def test_step_change_alarms_and_delays_stability(orc):
    """a step of 10·λ at round W/2 → not stable at round W.  By hand (δ = 0.005,
    λ = 0.25): 25 zeros give cum = min = −25δ; the 26th reward 2.5 makes n = 26,
    mean = 2.5/26, cum − min = 2.5 − 2.5/26 − δ ≈ 2.399 > λ → alarm at t = 25 and a reset;
    the constant 2.5 afterwards never alarms, so Exploitation begins at t = 25 + 50 = 75."""
    st = _stream(orc, _cfg(), [0.0] * 25 + [2.5] * 100)
    assert st["ph_alarms"] == 1
    assert st["first_exploit_t"] == 75 and st["phase"] == 1
    assert st["exploit_steps"] == 125 - 76


def test_alarm_threshold_hand_computed(orc):
    """Stream 0, 0, 0, 1 with δ = 0: after the 4th reward n = 4, mean = 1/4, cum = 3/4 and
    min = 0, so the detector alarms iff λ < 3/4 (exact in binary)."""
    for lam, alarms in ((0.5, 1), (0.74, 1), (0.75, 0), (0.8, 0)):
        st = _stream(orc, _cfg(ph_delta=0.0, ph_lambda=lam, ph_window=1000), [0.0, 0.0, 0.0, 1.0])
        assert st["ph_alarms"] == alarms, lam


def test_alarm_in_exploitation_reenters_exploration(orc):
    """drift after convergence re-enters Exploration with the detector reset."""
    st = _stream(orc, _cfg(ph_window=10), [0.1] * 30 + [2.0] + [0.1] * 5)
    assert st["first_exploit_t"] == 9 and st["ph_alarms"] >= 1 and st["phase"] == 0
    # steps 10..30 were greedy; after the alarm at t = 30 the detector needs 10 quiet rounds again
    assert st["exploit_steps"] == 21


def test_exploitation_is_eq2_greedy(orc):
    """Eq. 2: with W = 1 and λ = ∞ the tuner is in Exploitation from step 1 on; step 0
    with α > 0 picks the same arm as α = 0 (all fresh arms score α‖x‖ resp. 0 → lowest arm),
    so the whole run must equal the α0 = 0 run bit for bit (full synthetic environment)."""
    base = named_config("C2")
    base.update(T=800)
    ph = dict(base, ph_enable=1, ph_window=1, ph_lambda=1e300)
    st_ph, arms_ph, _ = orc.run_tuner(ph, orc.make_tuner(0, 1.0), T=800)
    st_g, arms_g, _ = orc.run_tuner(base, orc.make_tuner(0, 0.0), T=800)
    assert st_ph["first_exploit_t"] == 0 and st_ph["exploit_steps"] == 799
    for f in ("traj_hash", "sum_edp", "sum_reward", "n_active", "n_pruned_hist"):
        assert st_ph[f] == st_g[f], f
    assert np.array_equal(arms_ph["b"], arms_g["b"]) and np.array_equal(arms_ph["n"], arms_g["n"])


def test_never_stable_equals_disabled(orc):
    """λ = ∞ and W beyond T: the detector never switches, so the run is the §8(a) hot path."""
    base = named_config("C2")
    base.update(T=600)
    st_off, _, _ = orc.run_tuner(base, orc.make_tuner(5, 0.7), T=600)
    st_on, _, _ = orc.run_tuner(dict(base, ph_enable=1, ph_window=10**9, ph_lambda=1e300),
                                orc.make_tuner(5, 0.7), T=600)
    assert st_on["exploit_steps"] == 0 and st_on["first_exploit_t"] == NEVER and st_on["ph_alarms"] == 0
    for f in ("traj_hash", "sum_edp", "sum_reward", "sum_energy", "n_active"):
        assert st_on[f] == st_off[f], f


def test_default_detector_on_the_synthetic_environment(orc):
    """SPEC's defaults on C2's fluctuating trace: the detector does switch (the paper reports
    convergence at round 231, P:503 — order of magnitude only), alarms recur with the load,
    and exploit_steps is consistent with the phase history."""
    cfg = dict(named_config("C2"), ph_enable=1)
    st, _, _ = orc.run_tuner(cfg, orc.make_tuner(0, 1.0), T=4500)
    assert st["first_exploit_t"] != NEVER and st["first_exploit_t"] < 4500
    assert st["ph_alarms"] >= 1
    assert 0 < st["exploit_steps"] < 4500 - st["first_exploit_t"]
