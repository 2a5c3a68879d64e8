"""Pins of the oracle's ENV-S discrete-event server (ENV.md §7; SPEC inference_sim S:454-563;
PAPER P:129-131 continuous batching), independent of the CUDA path.  SPEC's worked examples
(S:512-516), closed forms of single requests, the conservation / KV-accounting invariants
(S:523-524), monotone physics and head-of-line admission under KV pressure."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from agft_inputs import named_config

W = 0.8


def _cfg(**kw):
    c = named_config("C2")
    c.update(kw)
    return c


def _dec(c, F):
    f = F / 1000.0
    return c["c_d"] / (c["beta"] + ((1.0 - c["beta"]) * (f / (c["f_max_hw_mhz"] / 1000.0))))


def test_single_request_spec_example():
    """empty queue, one request (ctx = 100, gen = 1, no cache) at f_max → one prefill
    iteration, then one decode iteration; prefill counter 100, decode 1."""
    c = _cfg()
    s = oracle.DesServer(c)
    assert s.push(0.0, 100, 1, 7)
    o = s.run(1800, W)
    waiting, running, prefill, decode, iters, kv, hits, misses = s.snap
    assert (waiting, running, prefill, decode, iters, kv, hits, misses) == (0, 0, 100, 1, 2, 0, 0, 1)
    # closed form (Fractions of the doubles, tolerance of a few roundings)
    pre = Fraction(c["c_p"]) / Fraction(1.8)
    dt0 = Fraction(oracle.DES_OVER) + 100 * pre
    dt1 = Fraction(oracle.DES_OVER) + Fraction(_dec(c, 1800))
    assert abs(Fraction(o["ttft"]) - (dt0 + dt1)) < Fraction(1, 10 ** 15)
    assert o["tpot"] == pytest.approx(float(dt1), rel=1e-15)        # one token, produced by the decode iteration
    busy = float(dt0 + dt1)
    f = 1.8
    pw = c["k_lin"] * f + c["k_cube"] * f * f * f
    ue = max(busy / W, c["u_floor"])
    assert o["E"] == pytest.approx((c["p_idle"] + pw * ue) * W, rel=1e-14)


def test_gen3_closed_form_and_retirement():
    c = _cfg()
    s = oracle.DesServer(c)
    s.push(0.0, 200, 3, 1)
    o = s.run(1200, W)
    pre = c["c_p"] / 1.2
    dt0 = oracle.DES_OVER + 200 * pre
    dd = oracle.DES_OVER + _dec(c, 1200)
    assert s.snap == [0, 0, 200, 3, 4, 0, 0, 1]
    assert o["ttft"] == pytest.approx(dt0 + dd, rel=1e-14)
    assert o["tpot"] == pytest.approx(dd, rel=1e-14)


def test_prefix_cache_spec_example():
    """two requests sharing a template with a warm prefix → the second's prefill is
    ctx − ⌊ctx/2⌋ (ENV.md §7: a cached template skips half the prompt); cache_hits increments."""
    c = _cfg()
    s = oracle.DesServer(c)
    s.push(0.0, 301, 5, 42)
    s.run(1500, W)
    assert s.snap[2] == 301 and s.snap[6:] == [0, 1]
    s.push(0.9, 301, 5, 42)
    s.run(1500, 2 * W)
    assert s.snap[2] == 301 - 150 and s.snap[6:] == [1, 0]
    s.push(1.7, 301, 5, 43)                                           # a new template misses again
    s.run(1500, 3 * W)
    assert s.snap[2] == 301 and s.snap[6:] == [0, 1]


def test_idle_and_busy_window_energy_spec():
    """idle window → energy = p_idle·W; busy window at u = 1, f = 1.8 GHz with p_idle = 60,
    k_lin = 80, k_cube = 15 → P = 291.48 W, energy 233.184 J."""
    c = _cfg(p_idle=60.0, k_lin=80.0, k_cube=15.0)
    s = oracle.DesServer(c)
    o = s.run(1800, W)
    assert o["E"] == pytest.approx(60.0 * W, rel=1e-15) and o["ttft"] == 0.0
    assert o["tpot"] == pytest.approx(_dec(c, 1800), rel=1e-15) and s.snap == [0] * 8
    s = oracle.DesServer(c)
    for i in range(60):                                               # long prompts keep it busy past W
        s.push(W + 1e-3 * i, 8000, 50, 100 + i)
    o = s.run(1800, 2 * W)
    assert o["E"] == pytest.approx(233.184, rel=1e-12)


def _run_windows(c, reqs, F, n_win):
    s = oracle.DesServer(c)
    out, snaps, states = [], [], []
    for t in range(n_win):
        for (arr, ctx, gen, tm) in reqs:
            if t * W <= arr < (t + 1) * W:
                s.push(arr, ctx, gen, tm)
        out.append(s.run(F, (t + 1) * W))
        snaps.append(s.snap)
        states.append(s.state)
    return out, snaps, states


def _requests(rng, n, ctx_rng, gen_rng, rate, pool=500):
    t = 0.0
    reqs = []
    for _ in range(n):
        t += rng.exponential(1.0 / rate)
        reqs.append((t, int(rng.integers(*ctx_rng)), int(rng.integers(*gen_rng)), int(rng.integers(0, pool))))
    return reqs


def test_conservation_and_kv_accounting():
    """Σ window decode counters = Σ tokens generated (finished requests contribute
    gen, running ones their tokens so far); the incremental KV usage equals the usage recomputed
    from the live requests after every window."""
    c = _cfg()
    rng = np.random.default_rng(5)
    reqs = _requests(rng, 400, (256, 1025), (20, 351), rate=6.0)
    n_win = 120
    out, snaps, states = _run_windows(c, reqs, 1200, n_win)
    st = states[-1]
    pushed = [r for r in reqs if r[0] < n_win * W]
    assert st["dropped"] == 0
    admitted = pushed[: len(pushed) - st["qlen"]]                       # FIFO: the queue holds the latest
    produced = sum(r[2] for r in admitted) - sum(gen - d for (ctx, gen, d, p) in st["running"])
    assert sum(sn[3] for sn in snaps) == produced
    for sn, stt in zip(snaps, states):
        assert sn[5] == stt["kv"] == sum(ctx + gen for (ctx, gen, d, p) in stt["running"])
        assert sn[1] == stt["nrun"] == len(stt["running"])
        assert all(d < gen for (ctx, gen, d, p) in stt["running"])


def test_fifo_head_of_line_under_kv_pressure():
    """Admission is FIFO while the KV footprint fits: with room for one 600-token request
    a second waits (counted in `waiting`) until the first retires, even if a smaller third fits."""
    c = _cfg(kv_total=1000)
    s = oracle.DesServer(c)
    s.push(0.0, 500, 100, 1)
    s.push(0.01, 500, 100, 2)                                         # would need 1200 > 1000
    s.push(0.02, 100, 10, 3)                                          # would fit, but is behind it
    s.run(1800, 0.05)
    assert s.snap[0] == 2 and s.snap[1] == 1 and s.snap[5] == 600
    assert not s.push(0.06, 900, 200, 4)                              # can never fit: dropped
    assert s.state["dropped"] == 1


@pytest.mark.parametrize("ctx,gen", [(100, 1), (2000, 20), (6000, 5)])
def test_raising_f_never_increases_ttft(ctx, gen):
    """S:526 monotone physics, single request: TTFT and every iteration are non-increasing in f."""
    c = _cfg()
    prev = None
    for F in range(210, 1801, 15):
        s = oracle.DesServer(c)
        s.push(0.0, ctx, gen, 0)
        o = s.run(F, 40 * W)
        if prev is not None:
            assert o["ttft"] <= prev
        prev = o["ttft"]


def test_long_generation_vs_long_context_ttft():
    """at a fixed clock, Long Generation's TTFT < Long Context's (500 requests, same seed)."""
    c = _cfg()
    res = {}
    for name, ctx_rng, gen_rng in (("lg", (1, 257), (350, 351)), ("lc", (1024, 8193), (1, 101))):
        rng = np.random.default_rng(11)
        reqs = _requests(rng, 500, ctx_rng, gen_rng, rate=2.9)
        n_win = int(reqs[-1][0] / W) + 200
        out, snaps, _ = _run_windows(c, reqs, 1305, n_win)
        w = [o["ttft"] for o, sn in zip(out, snaps) if o["ttft"] > 0]
        res[name] = float(np.mean(w))
    assert res["lg"] < res["lc"]


def test_closed_loop_tuner_runs_on_the_server():
    """cl_enable = 2: every decision reads the last window's snapshot (ENV.md §7); the run is
    deterministic, EDP stays positive, the base sums stay 0 (no f_max server)."""
    c = _cfg(cl_enable=2, T=600)
    tu = oracle.tuner_from(c)
    st1, arms1, rec1 = oracle.run_tuner(c, tu, T=600, record=True)
    st2, _, _ = oracle.run_tuner(c, tu, T=600)
    assert st1["traj_hash"] == st2["traj_hash"] and st1["sum_edp"] == st2["sum_edp"]
    assert st1["steps"] == 600 and st1["base_energy"] == 0.0 and st1["base_edp"] == 0.0
    assert np.all(rec1["edp"] > 0) and np.all(np.isfinite(rec1["edp"]))
    x = rec1["x"].reshape(600, -1)
    assert np.all(x[0] == 0.0) and np.all((x >= 0) & (x <= 1))
    # the server's load responds to the clock: at the lowest clock the queue builds up
    low = dict(c, n_arms=1, prune_enable=0)
    hi = dict(c, n_arms=1, prune_enable=0, f_min_mhz=1800)
    sl, _, rl = oracle.run_tuner(low, oracle.tuner_from(low), T=600, record=True)
    sh, _, rh = oracle.run_tuner(hi, oracle.tuner_from(hi), T=600, record=True)
    assert sl["sum_ttft"] > sh["sum_ttft"]


def test_window_arrivals_follow_the_trace():
    """ENV.md §7: window t queues the ENV-T row's a = hits + misses arrivals, evenly spaced, with
    lengths from the window's prototype."""
    c = _cfg()
    s = oracle.DesServer(c)
    rows = oracle.trace_rows(c, 0, 0, 50)
    arrived = 0
    for t in range(50):
        s.window(0, t, 1305)
        arrived += int(rows[t][6] + rows[t][7])
        st = s.state
        assert st["qlen"] + st["nrun"] + st["dropped"] <= arrived
    assert arrived > 0
