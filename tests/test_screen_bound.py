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
