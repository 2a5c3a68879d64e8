"""The historical-pruning screen of the SEG kernels (seg_common.cuh::hist_screen_safe) may skip the
exact canonical-tree evaluation of ENV.md §4.8 only when that evaluation would remove nothing.  This
replays the screen's arithmetic on the host (IEEE binary64, the same operation order; the device may
contract a product into an FMA, which only tightens the rounding) and checks the claim against the
exact pruning threshold computed as the oracle computes it (oracle.tree128 canonical sums), on random
and adversarial mean sets: near-threshold outliers, large mean / spread ratios (cancellation), ties,
two-arm sets and every k_h of the C4 sweep."""
import numpy as np
import pytest

import oracle

U = 2.0 ** -53


def screen_safe(vals, kh):
    """Host replay of hist_screen_safe (any summation order is covered by its bound)."""
    v = np.asarray(vals, np.float64)
    mn, mx = float(v.min()), float(v.max())
    if not mx > mn:
        return True
    s1 = 0.0
    s2 = 0.0
    for e in v:
        s1 += float(e)
        s2 += float(e) * float(e)
    inq = 1.0 / len(v)
    m2, mu = s2 * inq, s1 * inq
    V = m2 - mu * mu
    dV = 64.0 * U * m2
    if not V - dV > 0.0:
        return False
    sd_lo = np.sqrt(V - dV) * (1.0 - 8.0 * U)
    thr_lo = (mn + kh * sd_lo) * (1.0 - 16.0 * U)
    return mx < thr_lo


def exact_removes(vals, keys, kh):
    """ENV.md §4.8 as the oracle evaluates it: μ and σ from the canonical 128-slot tree."""
    slots = np.zeros(128)
    slots[keys] = vals
    nq = float(len(vals))
    mu = oracle.tree128(slots) / nq
    d2 = np.zeros(128)
    d2[keys] = [(e - mu) * (e - mu) for e in vals]
    sd = np.sqrt(oracle.tree128(d2) / nq)
    thr = float(np.min(vals)) + kh * sd
    return bool(np.any(np.asarray(vals) > thr)), thr


def _cases(rng):
    for _ in range(3000):                               # random sets
        n = int(rng.integers(2, 33))
        base = float(rng.lognormal(0.0, 2.0))
        yield base * rng.lognormal(0.0, float(rng.choice([1e-9, 1e-6, 1e-3, 0.1, 1.0])), n)
    for _ in range(1500):                               # one outlier placed at the exact threshold ± ulps
        n = int(rng.integers(2, 33))
        v = float(rng.lognormal(0, 1)) * (1 + 1e-3 * rng.standard_normal(n))
        yield v
    for _ in range(300):                                # large mean, tiny spread (cancellation in Σe² − nμ²)
        n = int(rng.integers(2, 33))
        yield 1e6 + rng.standard_normal(n) * float(rng.choice([1e-4, 1e-2, 1.0]))
    yield np.array([2.0, 2.0, 2.0])
    yield np.array([2.0, 2.1, 5.0])                     # S:293-295 (σ = 1.3912)


@pytest.mark.parametrize("kh", [0.0, 0.5, 1.0, 2.0, 4.0])
def test_screen_never_skips_a_removal(kh):
    rng = np.random.default_rng(int(kh * 10) + 7)
    safe_count = 0
    for vals in _cases(rng):
        vals = np.abs(np.asarray(vals, np.float64)) + 1e-300
        keys = np.sort(rng.choice(128, size=len(vals), replace=False))
        removes, thr = exact_removes(vals, keys, kh)
        # adversarial: move the largest mean onto the exact threshold and its neighbours
        for probe in (None, -2, -1, 0, 1, 2):
            v = vals.copy()
            if probe is not None:
                j = int(np.argmax(v))
                t = thr
                for _ in range(abs(probe)):
                    t = np.nextafter(t, np.inf if probe > 0 else -np.inf)
                if t <= float(np.min(np.delete(v, j))):
                    continue
                v[j] = t
            rm, _ = exact_removes(v, keys, kh)
            if screen_safe(v, kh):
                safe_count += 1
                assert not rm, (kh, v.tolist())
    if kh > 2.0:                                        # k_h ≤ 2 prunes any distinct set (Popoviciu: σ ≤ range/2)
        assert safe_count > 100                         # the screen decides the easy cases


# ---- the incremental screen (seg_common.cuh::ScreenCache): after a safe full screen, the cached bound
# is reused while Q's membership is unchanged and its means move (D ≥ Σ|Δē|, M = max moved mean)

def screen_full_cache(vals, kh):
    """Host replay of hist_screen_full: (safe, cache) with the device's operation order."""
    v = np.asarray(vals, np.float64)
    n = len(v)
    mn, mx = float(v.min()), float(v.max())
    c = {"ok": False, "mx": mx, "D": 0.0, "M": -np.inf,
         "B": (1.0 + kh * (1.0 / np.sqrt(float(n)))) * (1.0 + 8.0 * U)}
    if not mx > mn:
        c["P"] = mn
        c["ok"] = kh >= 0.0
        return True, c
    s1 = 0.0
    s2 = 0.0
    for e in v:
        s1 += float(e)
        s2 += float(e) * float(e)
    inq = 1.0 / n
    m2, mu = s2 * inq, s1 * inq
    V = m2 - mu * mu
    dV = 64.0 * U * m2
    if not V - dV > 0.0:
        return False, c
    sd_lo = np.sqrt(V - dV) * (1.0 - 8.0 * U)
    c["P"] = mn + kh * sd_lo
    safe = mx < c["P"] * (1.0 - 16.0 * U)
    c["ok"] = bool(safe and kh >= 0.0)
    return safe, c


def inc_safe(c):
    R = (c["P"] * (1.0 - 8.0 * U) - c["D"] * c["B"]) * (1.0 - 20.0 * U)
    return c["ok"] and max(c["mx"], c["M"]) < R


def note(c, d, e):
    c["D"] = (c["D"] + d) * (1.0 + 8.0 * U)
    c["M"] = max(c["M"], e)


@pytest.mark.parametrize("kh", [0.5, 1.0, 2.0, 3.0, 4.0])
def test_incremental_screen_never_skips_a_removal(kh):
    """Random walks of the means of Q after a safe full screen (the device's per-step moves: one mean
    at a time, drifting toward the threshold, jumping, shrinking toward the minimum): whenever the
    cached bound says safe, the exact evaluation on the current means removes nothing."""
    rng = np.random.default_rng(int(kh * 100) + 11)
    used = 0
    for case in range(1500):
        n = int(rng.integers(2, 33))
        base = float(rng.lognormal(0.0, 1.5))
        vals = base * rng.lognormal(0.0, float(rng.choice([1e-6, 1e-3, 0.05, 0.3])), n)
        keys = np.sort(rng.choice(128, size=n, replace=False))
        safe, c = screen_full_cache(vals, kh)
        if not safe:
            continue
        _, thr = exact_removes(vals, keys, kh)
        gap = thr - float(vals.max())
        for step in range(60):
            j = int(rng.integers(n))
            mode = rng.integers(4)
            old = float(vals[j])
            if mode == 0:                                   # drift the largest toward the threshold
                j = int(np.argmax(vals))
                old = float(vals[j])
                new = old + abs(gap) * float(rng.uniform(0.0, 0.6))
            elif mode == 1:                                 # drop the minimum
                j = int(np.argmin(vals))
                old = float(vals[j])
                new = old - abs(gap) * float(rng.uniform(0.0, 0.3))
            elif mode == 2:                                 # tiny Welford-like move
                new = old * (1.0 + float(rng.normal(0.0, 1e-3)))
            else:                                           # collapse toward the mean (σ shrinks)
                new = old + (float(vals.mean()) - old) * float(rng.uniform(0.0, 1.0))
            if not new > 0.0:
                continue
            vals[j] = new
            note(c, abs(new - old), new)
            if inc_safe(c):
                used += 1
                rm, _ = exact_removes(vals, keys, kh)
                assert not rm, (kh, case, step, vals.tolist())
    if kh > 2.0:                                            # (k_h ≤ 2 prunes any distinct set, as above)
        assert used > 100                                   # the cache decides the easy steps
