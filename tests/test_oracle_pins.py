"""Pins of the CPU oracle against what the paper, SPEC's worked examples and the
mathematics fix — never against the oracle itself and never against the CUDA path.

Each test names the passage it pins (P:n = PAPER.md line, S:n = SPEC.md line).
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from agft_inputs import named_config, frequencies

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def cfg_small(**kw):
    c = named_config("C2")
    c.update(kw)
    return c


# ----------------------------------------------------------------- ENV.md §1 Philox
def test_philox_known_answers(orc):
    """Random123 Philox4x32-10 KATs (SURVEY §8(c) a0/a7 noise)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(t, 16) for t in line.split()]
        out = orc.philox(v[0:4], v[4:6])
        assert out.tolist() == v[6:10]
        n += 1
    assert n == 3


# ----------------------------------------------------------------- a2 context (§4.1)
def _row(waiting=0, running=0, prefill=0, decode=0, iters=0, kv_used=0, hits=0, misses=0,
         noise=(0, 0, 0, 0)):
    return np.array([waiting, running, prefill, decode, iters, kv_used, hits, misses, *noise],
                    dtype=np.uint32)


def test_context_worked_example(orc):
    """800/80 tokens, 0.8 s, 40 iterations, 9 hits/1 miss → x2=1000, x3=100, x4=22, x7=0.9.
    Bounds are powers of two so the normalisation is exact and can be undone."""
    c = cfg_small(norm_lo=[0.0] * 7, norm_hi=[1.0, 2048.0, 2048.0, 64.0, 64.0, 1.0, 1.0])
    x = orc.context(c, _row(prefill=800, decode=80, iters=40, hits=9, misses=1))
    assert x[1] * 2048.0 == 1000.0
    assert x[2] * 2048.0 == 100.0
    assert x[3] * 64.0 == 22.0
    assert x[6] == 0.9
    assert x[0] == 0.0


def test_context_empty_window_is_zero(orc):
    """the all-zero window gives the zero vector; zero denominators are safe."""
    x = orc.context(cfg_small(), _row())
    assert np.all(x == 0.0) and np.all(np.isfinite(x))


def test_normalize_examples(orc):
    """1000 on (0,2000) → 0.5; below lo → 0; above hi → 1; lo = hi → 0."""
    c = cfg_small(norm_lo=[0.0] * 7, norm_hi=[1.0, 2000.0, 1.0, 1.0, 1.0, 1.0, 1.0])
    assert orc.context(c, _row(prefill=800))[1] == 0.5            # 800/0.8 = 1000
    c2 = cfg_small(norm_lo=[0.0, 5000.0] + [0.0] * 5, norm_hi=[1.0, 6000.0] + [1.0] * 5)
    assert orc.context(c2, _row(prefill=800))[1] == 0.0           # below lo
    assert orc.context(c2, _row(prefill=8000))[1] == 1.0          # above hi
    c3 = cfg_small(norm_lo=[0.0, 7.0] + [0.0] * 5, norm_hi=[1.0, 7.0] + [1.0] * 5)
    assert orc.context(c3, _row(prefill=8000))[1] == 0.0          # lo = hi


def test_context_bounds_property(orc):
    """x6, x7 ∈ [0,1] and every x finite for any snapshot."""
    rng = np.random.default_rng(0)
    c = cfg_small()
    for _ in range(500):
        r = _row(*rng.integers(0, 100000, 8))
        r[5] = min(r[5], c["kv_total"])
        x = orc.context(c, r)
        assert np.all(np.isfinite(x)) and np.all((x >= 0) & (x <= 1))


# ----------------------------------------------------------------- a7 ENV-R (ENV.md §3)
def _rec_cfg(**kw):
    c = cfg_small(p_idle=60.0, k_lin=80.0, k_cube=15.0, W=0.8, u_floor=0.0, c_d=0.01, beta=0.67)
    c.update(kw)
    return c


def test_power_worked_example(orc):
    """p_idle=60, k_lin=80, k_cube=15, f=1.8 GHz, u=1 → P=291.48 W, E=233.184 J.
    A busy window (u ≥ 1 saturates the power term) with zero noise (nE = 1)."""
    c = _rec_cfg()
    # iters=100 at c_d=0.01 s → 1.0 s of decode > W: u ≥ 1; noise words chosen so nE = nT = 1:
    # u53 = 0.5 exactly when the 53-bit mantissa word is 2^52 → a = 2^31, b = 0.
    row = _row(running=10, iters=100, decode=1000, noise=(1 << 31, 0, 1 << 31, 0))
    E, tpot, ttft, edp = orc.env_response(c, row, 1800)
    assert E == pytest.approx(233.184, rel=1e-12)
    assert E / 0.8 == pytest.approx(291.48, rel=1e-12)
    assert edp == E * tpot


def test_power_idle_window(orc):
    """an idle window consumes p_idle × W (with no utilisation floor)."""
    c = _rec_cfg()
    E, tpot, ttft, edp = orc.env_response(c, _row(noise=(1 << 31, 0, 1 << 31, 0)), 900)
    assert E == 60.0 * 0.8
    # idle: q = 1, g = 1 → TPOT is the bare decode time per iteration at 900 MHz (S:477 form)
    f, fmax = 0.9, 1.8
    assert tpot == pytest.approx(0.01 / (0.67 + 0.33 * f / fmax), rel=1e-15)


def test_response_monotone_physics():
    """SPEC inference_sim invariants: at a fixed window, raising f never raises
    TTFT/TPOT and strictly raises power when busy; EDP is finite and positive."""
    import oracle as orc
    c = named_config("C2")
    rows = orc.trace_rows(c, 3, 0, 200)
    for row in rows[::7]:
        prev = None
        for F in range(210, 1801, 15):
            E, tpot, ttft, edp = orc.env_response(c, row, F)
            assert edp > 0 and math.isfinite(edp)
            if prev:
                assert tpot <= prev[1] * (1 + 1e-15) and ttft <= prev[2] * (1 + 1e-15)
            prev = (E, tpot, ttft)


def test_edp_u_shape_per_prototype(orc):
    """§3.2 'U-shaped' EDP curves with interior argmins in the paper's bands
    (SURVEY calibration target; S:537 ≥10% below both endpoints)."""
    base = named_config("C2")
    argmins = []
    for p in range(5):
        w = [0] * 5
        w[p] = 256
        c = dict(base, weight=w)
        rows = orc.trace_rows(c, 11, 0, 600)
        freqs = list(range(210, 1801, 15))
        curve = [np.mean([orc.env_response(c, r, F)[3] for r in rows]) for F in freqs]
        k = int(np.argmin(curve))
        assert 0 < k < len(freqs) - 1
        assert curve[k] < 0.9 * curve[0] and curve[k] < 0.97 * curve[-1]
        argmins.append(freqs[k])
    # ordering of the paper's Table 6 offline column: compute-heavy ≥ efficiency
    normal, longctx, longgen, highconc, hithit = argmins
    assert longctx >= normal and highconc >= normal and longctx >= hithit
    assert all(1100 <= f <= 1500 for f in argmins), argmins


# ----------------------------------------------------------------- a8 EDP / reward
def test_edp_and_reward_examples(orc):
    """S:402-404 EDP products; S:412-413 reward zero / clip; bounded and monotone."""
    assert 130.0 * 2.0 == 260.0
    assert abs(129.058 * 0.0188 - 2.427) < 0.005            # Table 3 consistency (AMB-4)
    win = [1.0, 3.0, 2.0, 5.0, 4.0]                          # median 3
    assert orc.median(win) == 3.0
    assert orc.median([4.0, 1.0, 3.0, 2.0]) == 2.5            # even count: mean of middles
    assert orc.reward(3.0, win) == 0.0                        # edp = ref → 0
    assert orc.reward(9.0, win) == -2.0                       # edp = 3 ref → −2 (clipped)
    assert orc.reward(123.0, []) == 0.0                       # first window
    rs = [orc.reward(e, win) for e in np.linspace(0.0, 20.0, 101)]
    assert all(-2.0 <= r <= 2.0 for r in rs)
    assert all(a >= b for a, b in zip(rs, rs[1:]))            # non-increasing in EDP


# ----------------------------------------------------------------- reductions
def test_tree128_exact_on_integers(orc):
    rng = np.random.default_rng(1)
    for _ in range(50):
        v = rng.integers(-2**40, 2**40, 128).astype(np.float64)
        assert orc.tree128(v) == float(sum(int(a) for a in v))


def test_tree128_is_pairwise_not_sequential(orc):
    """The canonical order matters (AMB-26): 2^53 + 1 + 1 sequentially rounds to 2^53,
    pairwise (2^53 + 0) + (1 + 1) is exact."""
    v = np.zeros(128)
    v[0], v[2], v[3] = 2.0**53, 1.0, 1.0
    assert orc.tree128(v) == 2.0**53 + 2.0
    assert (2.0**53 + 1.0) + 1.0 == 2.0**53


# ----------------------------------------------------------------- linear algebra
def _frac_inverse(M):
    d = len(M)
    A = [[Fraction(M[i][j]) for j in range(d)] + [Fraction(int(i == j)) for j in range(d)]
         for i in range(d)]
    for c in range(d):
        p = next(r for r in range(c, d) if A[r][c] != 0)
        A[c], A[p] = A[p], A[c]
        pv = A[c][c]
        A[c] = [a / pv for a in A[c]]
        for r in range(d):
            if r != c and A[r][c] != 0:
                f = A[r][c]
                A[r] = [a - f * b for a, b in zip(A[r], A[c])]
    return [row[d:] for row in A]


def test_invert_and_solve_vs_exact_rationals(orc):
    rng = np.random.default_rng(2)
    for d in (1, 2, 4, 7):
        for _ in range(10):
            X = rng.integers(-8, 9, (d + 3, d)) / 8.0
            A = np.eye(d) + X.T @ X                  # exact: dyadic entries
            b = rng.integers(-16, 17, d) / 16.0
            inv = _frac_inverse(A.tolist())
            got = orc.invert(A)
            ex = np.array([[float(v) for v in r] for r in inv])
            assert np.allclose(got, ex, rtol=1e-12, atol=1e-14)
            th = orc.solve(A, b)
            exth = [float(sum(inv[i][j] * Fraction(b[j]) for j in range(d))) for i in range(d)]
            assert np.allclose(th, exth, rtol=1e-12, atol=1e-14)


def _core_cfg(K, d, **kw):
    c = cfg_small(n_arms=K, d=d, prune_enable=0, f_step_mhz=15)
    c.update(kw)
    return c


def test_update_fresh_arm_closed_form(orc):
    """fresh arm, x=e1, r=1 → A=diag(2,1,…), b=e1, θ=(½,0,…); r=0 → b=θ=0."""
    for d in (1, 4, 7):
        c = _core_cfg(1, d)
        x = np.zeros((1, d)); x[0, 0] = 1.0
        _, a, _ = orc.run_tuner(c, T=1, inject={"x": x, "reward": np.ones((1, 1))})
        A = np.eye(d); A[0, 0] = 2.0
        assert np.array_equal(a["A"][0], A)
        assert np.array_equal(a["b"][0], np.eye(d)[0])
        assert a["theta"][0][0] == 0.5 and np.all(a["theta"][0][1:] == 0)
        _, a, _ = orc.run_tuner(c, T=1, inject={"x": x * 0.75, "reward": np.zeros((1, 1))})
        assert np.all(a["b"][0] == 0) and np.all(a["theta"][0] == 0)


def test_sherman_morrison_closed_form(orc):
    """(I + x xᵀ)⁻¹ = I − x xᵀ / (1 + xᵀx): one update of a fresh arm."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        d = int(rng.integers(1, 8))
        x = rng.random((1, d))
        _, a, _ = orc.run_tuner(_core_cfg(1, d), T=1, inject={"x": x, "reward": np.zeros((1, 1))})
        xv = x[0]
        ex = np.eye(d) - np.outer(xv, xv) / (1.0 + xv @ xv)
        assert np.allclose(a["Ainv"][0], ex, rtol=1e-13, atol=1e-15)


def test_exact_rational_bruteforce(orc):
    """North-star pin: d ≤ 4, ≤ 20 updates with dyadic inputs; A⁻¹ and θ exact via Fractions."""
    rng = np.random.default_rng(4)
    for trial in range(12):
        d = int(rng.integers(1, 5))
        T = int(rng.integers(1, 21))
        x = rng.integers(0, 9, (T, d)) / 8.0
        r = rng.integers(-16, 17, (T, 1)) / 8.0
        _, a, _ = orc.run_tuner(_core_cfg(1, d), T=T, inject={"x": x, "reward": r})
        A = [[Fraction(int(i == j)) for j in range(d)] for i in range(d)]
        b = [Fraction(0)] * d
        for t in range(T):
            for i in range(d):
                b[i] += Fraction(r[t, 0]) * Fraction(x[t, i])
                for j in range(d):
                    A[i][j] += Fraction(x[t, i]) * Fraction(x[t, j])
        inv = _frac_inverse(A)
        ex_inv = np.array([[float(v) for v in row] for row in inv])
        ex_th = np.array([float(sum(inv[i][j] * b[j] for j in range(d))) for i in range(d)])
        assert np.array_equal(a["A"][0], np.array([[float(v) for v in row] for row in A]))
        assert np.allclose(a["Ainv"][0], ex_inv, rtol=1e-12, atol=1e-15)
        assert np.allclose(a["theta"][0], ex_th, rtol=1e-12, atol=1e-14)


def test_ridge_equivalence_10k_updates(orc):
    """S:185 / S:747: after 10⁴ random updates θ equals (I+Σxxᵀ)⁻¹Σrx within 1e-9."""
    rng = np.random.default_rng(5)
    d, T = 7, 10000
    x = rng.random((T, d))
    r = rng.uniform(-2, 2, (T, 1))
    _, a, _ = orc.run_tuner(_core_cfg(1, d), T=T, inject={"x": x, "reward": r})
    A = np.eye(d) + x.T @ x
    b = x.T @ r[:, 0]
    th = np.linalg.solve(A, b)
    assert np.allclose(a["theta"][0], th, rtol=1e-9, atol=1e-12)
    ev = np.linalg.eigvalsh(a["Ainv"][0])
    assert np.all(ev > 0) and np.all(ev <= 1 + 1e-12)      # SPD, λ_min(A) ≥ 1


def test_d1_reduces_to_ridge_mean_ucb(orc):
    """d=1, x≡1: A = 1+n, θ = Σr/(1+n), score = Σr/(1+n) + α/√(1+n) (textbook UCB form)."""
    K, T = 3, 12
    rng = np.random.default_rng(6)
    c = _core_cfg(K, 1, tau=1e300)                          # α_t ≡ α0
    rew = rng.integers(-8, 9, (T, K)) / 8.0
    x = np.ones((T, 1))
    _, a, rec = orc.run_tuner(c, orc.tuner_from(c, alpha0=0.75), T=T,
                              inject={"x": x, "reward": rew}, record=True, scores=True)
    n = np.zeros(K); sr = np.zeros(K)
    for t in range(T):
        ex = sr / (1 + n) + 0.75 / np.sqrt(1 + n)
        assert np.allclose(rec["scores"][t], ex, rtol=1e-14)
        k = int(rec["arm"][t])
        assert k == int(np.argmax(ex))
        n[k] += 1; sr[k] += rew[t, k]


def test_select_examples(orc):
    """fresh arms tie → lowest frequency. S:164: arm A after (e1, r=1), arm B fresh,
    ctx = e1, α = 0 → A (0.5 vs 0)."""
    c = _core_cfg(4, 3)
    x = np.array([[0.3, 0.2, 0.1]])
    _, _, rec = orc.run_tuner(c, T=1, inject={"x": x}, record=True)
    assert rec["arm"][0] == 0
    c2 = _core_cfg(2, 3)
    e1 = np.array([[1.0, 0, 0], [1.0, 0, 0]])
    follow = np.array([0, orc.FREE], np.uint8)               # force A at t=0, free at t=1
    _, _, rec = orc.run_tuner(c2, orc.tuner_from(c2, alpha0=0.0), T=2, follow=follow,
                              inject={"x": e1, "reward": np.array([[1.0, 0.0], [0.0, 0.0]])},
                              record=True, scores=True)
    assert rec["scores"][1].tolist() == [0.5, 0.0] and rec["arm"][1] == 0


def test_exact_tie_constructor_is_flagged(orc):
    """Arm 0 after (e1, r=1) scores ½ + α/√2; fresh arm 1 scores α: tied at
    α = ½/(1 − 1/√2) ≈ 1.7071 — the step must be flagged as a near-tie (AMB-6)."""
    c = _core_cfg(2, 2, tau=1e300)
    alpha = 0.5 / (1.0 - 1.0 / math.sqrt(2.0))
    e1 = np.array([[1.0, 0.0], [1.0, 0.0]])
    follow = np.array([0, orc.FREE], np.uint8)
    _, _, rec = orc.run_tuner(c, orc.tuner_from(c, alpha0=alpha), T=2, follow=follow,
                              inject={"x": e1, "reward": np.array([[1.0, 0.0], [0.0, 0.0]])},
                              record=True, scores=True)
    assert abs(rec["scores"][1][0] - rec["scores"][1][1]) < 1e-15
    assert rec["near_tie"][1] == 1
    # away from the tie nothing is flagged
    _, _, rec = orc.run_tuner(c, orc.tuner_from(c, alpha0=alpha * 1.01), T=2, follow=follow,
                              inject={"x": e1, "reward": np.array([[1.0, 0.0], [0.0, 0.0]])},
                              record=True)
    assert rec["near_tie"][1] == 0


def test_alpha_zero_is_greedy_and_scale_invariant(orc):
    """α=0 ≡ greedy (Eq. 2); scaling all rewards by 2^k keeps argmax."""
    rng = np.random.default_rng(7)
    K, d, T = 6, 4, 300
    c = _core_cfg(K, d)
    x = rng.random((T, d))
    rew = rng.uniform(-1, 1, (T, K))
    tu = orc.tuner_from(c, alpha0=0.0)
    _, _, r1 = orc.run_tuner(c, tu, T=T, inject={"x": x, "reward": rew}, record=True, scores=True)
    _, _, r2 = orc.run_tuner(c, tu, T=T, inject={"x": x, "reward": rew * 4.0}, record=True)
    assert np.array_equal(r1["arm"], r2["arm"])
    # greedy: the chosen arm maximises θ·x (scores at α=0 are θ·x)
    for t in range(T):
        s = r1["scores"][t]
        assert s[r1["arm"][t]] == np.nanmax(s)


def test_zero_context_picks_lowest_active(orc):
    """AMB-20: x = 0 → every score is exactly 0 → lowest active arm; A, b unchanged, n advances."""
    c = _core_cfg(5, 3)
    T = 6
    x = np.zeros((T, 3))
    _, a, rec = orc.run_tuner(c, T=T, inject={"x": x, "reward": np.full((T, 5), 0.5)}, record=True)
    assert np.all(rec["arm"] == 0) and np.all(rec["near_tie"] == 0)
    assert np.array_equal(a["A"][0], np.eye(3)) and np.all(a["b"][0] == 0) and a["n"][0] == T


def test_regret_vs_uniform_random(orc):
    """a 12-arm linear bandit over 2,000 rounds has ≤ 15% of uniform-random regret."""
    K, d, T = 12, 4, 2000
    c = _core_cfg(K, d, tau=1e300)
    ratios = []
    for seed in range(5):
        rng = np.random.default_rng(100 + seed)
        th = rng.uniform(-1, 1, (K, d))
        x = rng.random((T, d))
        mean = x @ th.T                                            # [T, K]
        rew = mean + rng.normal(0, 0.1, (T, K))
        _, _, rec = orc.run_tuner(c, orc.tuner_from(c, alpha0=0.5), T=T,
                                  inject={"x": x, "reward": rew}, record=True)
        best = mean.max(axis=1)
        regret = np.sum(best - mean[np.arange(T), rec["arm"]])
        uniform = np.sum(best - mean.mean(axis=1))
        ratios.append(regret / uniform)
    assert max(ratios) <= 0.15, ratios


# ----------------------------------------------------------------- a10 pruning (§4.3)
def _prune_cfg(K=4, **kw):
    c = _core_cfg(K, 2, prune_enable=1)
    c.update(kw)
    return c


def _run_forced(orc, c, seq, edp_of_arm=None, reward_of_arm=None, tu=None):
    T = len(seq)
    K = c["n_arms"]
    x = np.tile([0.5, 0.25], (T, 1))
    edp = np.ones((T, K)) if edp_of_arm is None else np.tile(edp_of_arm, (T, 1))
    rew = np.zeros((T, K)) if reward_of_arm is None else np.tile(reward_of_arm, (T, 1))
    return orc.run_tuner(c, tu, T=T, follow=np.array(seq, np.uint8),
                         inject={"x": x, "edp": edp, "reward": rew}, record=True)


def test_extreme_pruning_gates(orc):
    """t=40, n=3, r̄=−1.5 → pruned; n=2 → kept; t=70 → kept (60 / 3 / −1.2)."""
    c = _prune_cfg(K=4, f_min_mhz=1200)               # above ½ f_max: no cascade
    rew = [-1.5, 0.0, 0.0, 0.0]
    seq = [1] * 38 + [0, 0, 0]                        # third sample of arm 0 at t=40
    st, a, _ = _run_forced(orc, c, seq, reward_of_arm=rew)
    assert a["active"][0] == 0 and st["n_pruned_extreme"] == 1
    st, a, _ = _run_forced(orc, c, [1] * 39 + [0, 0], reward_of_arm=rew)       # n = 2
    assert a["active"][0] == 1 and st["n_pruned_extreme"] == 0
    st, a, _ = _run_forced(orc, c, [1] * 68 + [0, 0, 0], reward_of_arm=rew)    # t = 70
    assert a["active"][0] == 1


def test_historical_pruning_sigma_examples(orc):
    """ē {2.0, 2.1, 5.0} (n ≥ 6) → σ_pop ≈ 1.39 → 5.0 pruned; {2.0, 2.1} → 2.1
    pruned (σ = 0.05); an arm with n = 5 and ē = 100 is kept. P:388: t ≥ 30, n ≥ 6."""
    c = _prune_cfg(K=4, f_min_mhz=1200)
    edp = [2.0, 2.1, 5.0, 100.0]
    seq = [0, 1, 2] * 6 + [0] * 12 + [3] * 5           # t=18..29 arm 0; then arm 3 five times
    st, a, rec = _run_forced(orc, c, seq[:32], edp_of_arm=edp)
    assert rec["n_active"][29] == 4                     # nothing before t = 30
    assert rec["active_mask"][30][0] == 0b1011          # t=30: 5.0 pruned (σ ≈ 1.39)
    assert a["active"].tolist() == [1, 0, 0, 1]         # t=31: 2.1 pruned (σ = 0.05)
    assert st["n_pruned_hist"] == 2
    st, a, _ = _run_forced(orc, c, seq, edp_of_arm=edp)
    assert a["active"][3] == 1 and a["n"][3] == 5       # n = 5 < 6: kept
    # σ of {2, 2.1, 5} is the population std (1.3912), not the sample std (1.7039)
    assert np.std([2.0, 2.1, 5.0]) == pytest.approx(1.3912, abs=1e-4)


def test_cascade_examples(orc):
    """f_max=1800: pruning 600 MHz (< 900) removes all lower arms;
    1200 → no cascade; 225 → only 210 cascades."""
    c = _prune_cfg(K=107, f_min_mhz=210)
    f = frequencies(c)
    for fp, expect_removed in ((600, set(range(0, f.index(600)))), (1200, set()), (225, {0})):
        k = f.index(fp)
        rew = np.zeros(107); rew[k] = -2.0
        seq = [106] * 37 + [k, k, k]
        st, a, _ = _run_forced(orc, c, seq, reward_of_arm=rew)
        removed = {j for j in range(107) if not a["active"][j]}
        assert removed == expect_removed | {k}
        assert st["n_pruned_cascade"] == len(expect_removed)


def test_pruning_fuzz_invariants(orc):
    """pruned arms never chosen, cascade monotone, never empty,
    extreme never reappears (all removals permanent in the hot path, AMB-12)."""
    rng = np.random.default_rng(9)
    for trial in range(20):
        K = int(rng.integers(2, 40))
        c = _core_cfg(K, 3, prune_enable=1, f_min_mhz=210, f_step_mhz=15 * int(rng.integers(1, 4)))
        c["f_max_hw_mhz"] = max(1800, c["f_min_mhz"] + (K - 1) * c["f_step_mhz"])
        T = 200
        x = rng.random((T, 3))
        edp = rng.uniform(0.5, 5.0, (T, K))
        tu = orc.tuner_from(c, alpha0=float(rng.uniform(0, 3)), hist_k=float(rng.choice([0.5, 1, 2])),
                            ext_reward_threshold=float(rng.uniform(-1.5, -0.5)))
        _, _, rec = orc.run_tuner(c, tu, T=T, inject={"x": x, "edp": edp}, record=True)
        prev = (1 << K) - 1
        for t in range(T):
            m = sum(int(rec["active_mask"][t][w]) << (32 * w) for w in range(4))
            assert m != 0                                   # never empty
            assert m & ~prev == 0                           # permanent
            assert (prev >> int(rec["arm"][t])) & 1         # chosen arm was active
            prev = m


def test_grid_counts():
    """S:273-275 / P:257: (210,1800,15) → 107 arms; (210,240,15) → 3; (210,1800,30) → 54."""
    assert len(frequencies(named_config("C2"))) == 107
    assert frequencies(named_config("C2"))[-1] == 1800
    assert len(range(210, 241, 15)) == 3 and len(range(210, 1801, 30)) == 54


# ----------------------------------------------------------------- ENV-T shapes (Table 1)
def test_trace_invariants_and_fingerprints(orc):
    """Table 1 + Fig. 7 qualitative fingerprints."""
    base = named_config("C2")
    cents = []
    for p in range(5):
        w = [0] * 5
        w[p] = 256
        c = dict(base, weight=w)
        rows = orc.trace_rows(c, 5, 0, 1500).astype(np.int64)
        wait, run, pre, dec, it, kv, hits, miss = rows[:, :8].T
        assert np.all(run <= c["cap"]) and np.all(kv <= c["kv_total"]) and np.all(hits >= 0)
        assert np.all(dec == run * it)
        xs = np.array([orc.context(c, r) for r in rows[::5].astype(np.uint32)])
        cents.append(xs.mean(axis=0))
    cents = np.array(cents)
    assert np.argmax(cents[:, 4]) == 3 and np.argmax(cents[:, 0]) == 3   # High Conc: x5, x1
    assert np.argmax(cents[:, 1]) == 1                                     # Long Context: x2
    assert np.argmax(cents[:, 6]) == 4 and cents[4, 6] > 0.8               # High Cache Hit: x7
    # Long Generation: gen fixed at 350 → KV per running request ≥ ctx_lo + 175
    c = dict(base, weight=[0, 0, 256, 0, 0])
    rows = orc.trace_rows(c, 5, 0, 300).astype(np.int64)
    run, kv = rows[:, 1], rows[:, 5]
    assert np.all(kv[run > 0] >= run[run > 0] * (1 + 175))


def test_arrivals_match_rate(orc):
    """Irwin–Hall arrivals: the mean count per window ≈ λ·W (Normal load, λ0 = 2.9)."""
    c = dict(named_config("C2"), weight=[256, 0, 0, 0, 0])
    rows = orc.trace_rows(c, 9, 0, 4000).astype(np.int64)
    a = rows[:, 6] + rows[:, 7]
    assert abs(a.mean() - 2.9 * 0.8) < 0.1


def test_determinism(orc):
    """byte-identical decisions across runs."""
    c = named_config("C2")
    s1, _, r1 = orc.run_tuner(c, T=800, record=True)
    s2, _, r2 = orc.run_tuner(c, T=800, record=True)
    assert s1 == s2 and np.array_equal(r1["arm"], r2["arm"])
