"""Round-2 pins of the oracle (VERDICT r1 "parity unpinned" items), each against something the
oracle does not compute itself: closed-form special values, a published hash test vector, a
hand derivation of the AMB-11 guard, and an exact-rational evaluation of one busy ENV-R window.

Citations: α_t = α0/√(1+t/τ) — PAPER.md:356 (Eq. 1, symbol α_t) read as SPEC.md:142, 214 (AMB-1);
the non-empty guard — SPEC.md:281 (AMB-11); the trajectory hash — FNV-1a 64 (ENV.md §4.9); ENV-R —
ENV.md §3.3 (the invented closed form, AMB-22; power form SPEC.md:472, decode form SPEC.md:477).
"""
from fractions import Fraction as Fr
import math

import numpy as np
import pytest

import oracle
from agft_inputs import named_config, with_overrides


def _inj_cfg(**kw):
    c = with_overrides(named_config("C2"), prune_enable=0, **kw)
    return c


# ------------------------------------------------------------------ a3: α_t at finite τ
@pytest.mark.parametrize("tau,alpha0", [(2.0, 1.5), (200.0, 1.0), (7.0, 0.3)])
def test_alpha_t_special_values_at_finite_tau(tau, alpha0):
    """A never-updated arm has A⁻¹ = I and θ = 0, so at context e1 its Eq. 1 score is exactly α_t.
    With α_t = α0/√(1+t/τ): t = 0 → α0; t = τ → α0/√2; t = 3τ → α0/2 (√4 = 2, exact);
    t = 8τ → α0/3 (√9 = 3, exact).  A 1-based t, a missing square root or α0/(1+t/τ) fails."""
    K, d = 16, 2
    ti = int(tau)
    T = 8 * ti + 1
    cfg = _inj_cfg(n_arms=K, d=d, tau=tau, T=T)
    x = np.zeros((T, d))
    x[:, 0] = 1.0
    reward = np.full((T, K), 2.0)          # the first arm stays ahead: every other arm stays fresh
    _, _, rec = oracle.run_tuner(cfg, oracle.make_tuner(0, alpha0), T=T, record=True, scores=True,
                                 inject={"x": x, "reward": reward})
    assert np.all(rec["arm"] == 0)
    s = rec["scores"]
    for t, want in ((0, alpha0), (3 * ti, alpha0 / 2.0), (8 * ti, alpha0 / 3.0)):
        assert np.all(s[t, 1:] == want), (t, s[t, 1:3], want)
    # t = τ: α0·(1/√2) to within one rounding of the division
    assert np.all(np.abs(s[ti, 1:] - alpha0 * math.sqrt(0.5)) <= 2 * np.spacing(alpha0))
    # and α_t is strictly decreasing in t for the fresh arms
    assert np.all(np.diff(s[:, 1]) < 0)


# ------------------------------------------------------------------ a10: AMB-11 non-empty guard
def _guard_run(r_arm1):
    """Three arms at 210/225/240 MHz (all below ½·f_max = 900 MHz, so any removal cascades to the
    lower arms); extreme pruning with n_E = 1; historical pruning off.  Forced pulls: arm 0 (r = −0.5),
    arm 1 (r = r_arm1), arm 2 (r = −2 < τ_E = −1.2).  At step 2 Ext = {2} and the cascade removes
    {0, 1}: the set would empty, so AMB-11 keeps the removed arm with the largest r̄, ties → lowest k."""
    K, d, T = 3, 2, 3
    cfg = with_overrides(named_config("C2"), n_arms=K, d=d, T=T, ext_round_limit=100, ext_min_samples=1,
                         hist_min_round=10**6, hist_min_samples=10**6)
    x = np.zeros((T, d))
    x[:, 0] = 1.0
    reward = np.zeros((T, K))
    reward[0, 0], reward[1, 1], reward[2, 2] = -0.5, r_arm1, -2.0
    follow = np.array([0, 1, 2], np.uint8)
    st, arms, rec = oracle.run_tuner(cfg, oracle.make_tuner(0, 1.0, -1.2, 1.0), T=T, follow=follow,
                                     record=True, inject={"x": x, "reward": reward})
    return st, arms, rec


def test_non_empty_guard_keeps_max_rbar_lowest_k_on_ties():
    st, arms, rec = _guard_run(-0.5)                  # r̄0 = r̄1 = −0.5: tie → arm 0 kept
    assert list(arms["active"]) == [1, 0, 0]
    assert st["n_pruned_extreme"] == 1 and st["n_pruned_cascade"] == 1 and st["n_pruned_hist"] == 0
    assert list(rec["n_active"]) == [3, 3, 1]


def test_non_empty_guard_keeps_the_max_rbar_arm():
    st, arms, _ = _guard_run(-0.3)                    # r̄1 = −0.3 > r̄0 = −0.5: arm 1 kept
    assert list(arms["active"]) == [0, 1, 0]
    assert st["n_pruned_extreme"] == 1 and st["n_pruned_cascade"] == 1


def test_guard_not_triggered_when_an_arm_survives():
    """Control: with a fourth arm above the cascade limit nothing is restored (arm 3 survives)."""
    K, d, T = 4, 2, 3
    cfg = with_overrides(named_config("C2"), n_arms=K, d=d, T=T, f_step_mhz=500, ext_round_limit=100,
                         ext_min_samples=1, hist_min_round=10**6, hist_min_samples=10**6)
    # arms at 210, 710, 1210, 1710 MHz: removing arm 1 (710 < 900) cascades to arm 0 only
    x = np.zeros((T, d))
    x[:, 0] = 1.0
    reward = np.zeros((T, K))
    reward[0, 0], reward[1, 2], reward[2, 1] = -0.5, 0.5, -2.0
    st, arms, _ = oracle.run_tuner(cfg, oracle.make_tuner(0, 1.0, -1.2, 1.0), T=T,
                                   follow=np.array([0, 2, 1], np.uint8), inject={"x": x, "reward": reward})
    assert list(arms["active"]) == [0, 0, 1, 1]
    assert st["n_pruned_extreme"] == 1 and st["n_pruned_cascade"] == 1


# ------------------------------------------------------------------ a11: FNV-1a trajectory hash
@pytest.mark.parametrize("text,want", [
    ("a", 0xaf63dc4c8601ec8c),          # FNV-1a 64 published test vectors (Fowler/Noll/Vo)
    ("foobar", 0x85944171f73967e8),
])
def test_trajectory_hash_is_fnv1a_64(text, want):
    """Chosen arms < 256 are hashed one octet per step, so forcing the arm sequence to the bytes of
    a string reproduces the published FNV-1a 64-bit hash of that string."""
    seq = np.frombuffer(text.encode(), np.uint8)
    T = len(seq)
    cfg = _inj_cfg(n_arms=128, d=2, T=T, f_min_mhz=210, f_step_mhz=12, f_max_hw_mhz=1800)
    x = np.zeros((T, 2))
    x[:, 0] = 1.0
    st, _, _ = oracle.run_tuner(cfg, oracle.make_tuner(0, 1.0), T=T, follow=seq, inject={"x": x})
    assert st["traj_hash"] == want
    assert st["last_arm"] == seq[-1]


def test_empty_trajectory_hash_is_the_offset_basis():
    st, _, _ = oracle.run_tuner(named_config("C1"), T=0)
    assert st["traj_hash"] == 0xcbf29ce484222325


# ------------------------------------------------------------------ a7: one busy ENV-R window
def _u53(a, b):
    return Fr(((a << 21) ^ (b >> 11)), 1 << 53)


def test_busy_window_against_exact_rationals():
    """ENV.md §3.3 for a window past the knee: 64 running + 192 waiting → ρ = 4, g = ρ√ρ = 8
    (exact); u > u_max, so q = u/(u_max(1−u_max)) (linear past the knee); u > 1 so the power
    saturates (ue = 1); TTFT has its waiting term.  The noise words give u53 = ½ → nT = nE = 1
    exactly.  Evaluated in exact rational arithmetic from the double constants; the oracle's
    correctly-rounded operation sequence must agree to a few ulp."""
    cfg = named_config("C2")
    waiting, running, prefill, decode, iters, kv, hits, misses = 192, 64, 20000, 64 * 40, 40, 1000, 3, 7
    N = [1 << 31, 0, 1 << 31, 0]
    assert _u53(N[0], N[1]) == Fr(1, 2)
    row = np.array([waiting, running, prefill, decode, iters, kv, hits, misses] + N, np.uint32)
    F = 1200
    E, TPOT, TTFT, EDP = oracle.env_response(cfg, row, F)

    c = {k: Fr(cfg[k]) for k in ("W", "p_idle", "k_lin", "k_cube", "u_floor", "u_max", "c_p", "c_d", "beta")}
    f = Fr(F, 1000)
    fmax = Fr(cfg["f_max_hw_mhz"], 1000)
    dec = c["c_d"] / (c["beta"] + (1 - c["beta"]) * (f / fmax))
    pre = c["c_p"] / f
    pw = c["k_lin"] * f + c["k_cube"] * f * f * f
    g = Fr(8)                                            # ρ = 256/64 = 4, ρ·√ρ = 8
    t_dec, t_pre = iters * dec, prefill * pre
    u = (t_dec + t_pre) * g / c["W"]
    assert u > 1                                         # past the knee and saturated
    q = u / (c["u_max"] * (1 - c["u_max"]))
    tpot = (dec + t_pre / iters) * g * q
    energy = (c["p_idle"] + pw * 1) * c["W"]
    ttft = (t_pre / (hits + misses) + t_dec * Fr(waiting, iters)) * q
    for got, want in ((E, energy), (TPOT, tpot), (TTFT, ttft), (EDP, energy * tpot)):
        assert abs(Fr(got) - want) <= abs(want) * Fr(1, 10**14), (got, float(want))


def test_medium_window_below_the_knee_against_exact_rationals():
    """The other branch: ρ ≤ 1 (g = 1), u ≤ u_max (q = 1/(1−u)), u above the floor."""
    cfg = named_config("C2")
    waiting, running, prefill, decode, iters, hits, misses = 0, 20, 3000, 20 * 30, 30, 1, 4
    N = [1 << 31, 0, 1 << 31, 0]
    row = np.array([waiting, running, prefill, decode, iters, 500, hits, misses] + N, np.uint32)
    F = 1500
    E, TPOT, TTFT, EDP = oracle.env_response(cfg, row, F)
    c = {k: Fr(cfg[k]) for k in ("W", "p_idle", "k_lin", "k_cube", "u_floor", "u_max", "c_p", "c_d", "beta")}
    f, fmax = Fr(F, 1000), Fr(cfg["f_max_hw_mhz"], 1000)
    dec = c["c_d"] / (c["beta"] + (1 - c["beta"]) * (f / fmax))
    pre = c["c_p"] / f
    pw = c["k_lin"] * f + c["k_cube"] * f * f * f
    t_dec, t_pre = iters * dec, prefill * pre
    u = (t_dec + t_pre) / c["W"]
    assert c["u_floor"] < u <= c["u_max"]
    q = 1 / (1 - u)
    tpot = (dec + t_pre / iters) * q
    energy = (c["p_idle"] + pw * u) * c["W"]
    ttft = (t_pre / (hits + misses)) * q
    for got, want in ((E, energy), (TPOT, tpot), (TTFT, ttft), (EDP, energy * tpot)):
        assert abs(Fr(got) - want) <= abs(want) * Fr(1, 10**14), (got, float(want))


# ------------------------------------------------------------------ a6: the recorded top-2 gap
def test_recorded_gap_matches_its_definition_on_a_hand_step():
    """ENV.md §4.5 gap on the exact-tie constructor's neighbourhood: after (e1, r = 1) on arm 0, at
    context e1 arm 0 scores ½ + α/√2 and the fresh arm 1 scores α.  At α = 1 the gap is
    (½ + 1/√2 − 1)/(½ + 1/√2) (arm 0 executed)."""
    K, d, T = 2, 2, 2
    cfg = _inj_cfg(n_arms=K, d=d, T=T, tau=1e300)
    x = np.zeros((T, d))
    x[:, 0] = 1.0
    reward = np.ones((T, K))
    _, _, rec = oracle.run_tuner(cfg, oracle.make_tuner(0, 1.0), T=T, record=True, scores=True,
                                 inject={"x": x, "reward": reward})
    assert rec["arm"][1] == 0
    s0 = 0.5 + math.sqrt(0.5)
    assert abs(rec["gap"][1] - (s0 - 1.0) / s0) < 1e-15
    assert rec["gap"][0] == 0.0 or rec["near_tie"][0] == 0   # step 0: two fresh arms, identical scores
