"""GPU parity of the offline sweep and regret (ENV.md §5) against
the CPU oracle: per-arm / per-prototype sums, window counts, per-window oracle arms and
sums bit-exact (ENV.md §0: same values, same left-to-right order); regret = the same
subtraction of bit-exact values."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from agft_inputs import named_config, tuner_params  # noqa: E402
from paper_2508_01744_b200 import AgftError, TunerBatch  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _gpu_sweep(cfg, T, chunks, ids=None, replay=False):
    params = tuner_params(cfg, ids)
    n = len(params["trace_id"])
    tb = TunerBatch(dict(cfg, n_tuners=n), params, device="cuda:0")
    sums = tb.new_sweep()
    bests = []
    t = 0
    for n_c in chunks:
        rec = tb.generate(t, n_c)
        bests.append(tb.sweep(rec, t, n_c, sums, best=True).cpu().numpy())
        if replay:
            tb.replay(rec, t, n_c)
        t += n_c
    assert t == T
    return tb, params, sums, np.concatenate(bests, axis=1)


def _check_trace(cfg, h, best, r, T):
    acc, b = oracle.sweep(cfg, r, 0, T, best=True)
    assert np.array_equal(h["S"][r], acc["S"]), "S"
    assert np.array_equal(h["SP"][r], acc["SP"]), "SP"
    assert np.array_equal(h["NP"][r], acc["NP"].astype(np.uint32)), "NP"
    assert np.array_equal(h["O"][r], acc["O"]), "O"
    assert np.array_equal(best[r], b), "k°"
    koff = [oracle.offline_arm(acc["SP"][p]) if acc["NP"][p] else 255 for p in range(5)]
    koff.append(oracle.offline_arm(acc["S"][:, 2]))
    return koff


def test_sweep_c2_chunked_bitexact():
    cfg = named_config("C2")
    tb, params, sums, best = _gpu_sweep(cfg, 4500, [1, 31, 968, 3500])
    tb.regret(sums)
    h = sums.host()
    koff = _check_trace(cfg, h, best, 0, 4500)
    assert list(h["koff"][0]) == koff


@pytest.mark.parametrize("kw", [dict(n_arms=1), dict(n_arms=128, f_step_mhz=12, f_min_mhz=210),
                                dict(n_arms=33, f_step_mhz=45), dict(d=2)])
def test_sweep_edge_grids(kw):
    cfg = dict(named_config("C3"), n_tuners=3, n_traces=3, **kw)
    tb, params, sums, best = _gpu_sweep(cfg, 777, [777])
    tb.regret(sums)
    h = sums.host()
    for r in range(3):
        assert list(h["koff"][r]) == _check_trace(cfg, h, best, r, 777)


def test_sweep_state_error_on_wrong_t0():
    cfg = named_config("C1")
    tb = TunerBatch(cfg, tuner_params(cfg), device="cuda:0")
    sums = tb.new_sweep()
    rec = tb.generate(0, 10)
    with pytest.raises(AgftError) as e:
        tb.sweep(rec, 5, 10, sums)
    assert e.value.code == -7
    tb.sweep(rec, 0, 10, sums)


def test_sweep_c4_full_size_sampled():
    """BASELINE configs[3] at full size: all 256 traces × 108,000 windows in 4,500-window
    chunks; sampled traces bit-exact, invariants on every trace."""
    cfg = named_config("C4")
    T = cfg["T"]
    tb, params, sums, best = _gpu_sweep(cfg, T, [4500] * (T // 4500), ids=list(range(256)))
    tb.regret(sums)
    h = sums.host()
    assert np.all(h["NP"].sum(axis=1) == T)
    assert np.all(h["O"][:, 0][:, None] <= h["S"][:, :, 2])
    for r in (0, 201):                                   # one diurnal, one burst trace
        assert list(h["koff"][r]) == _check_trace(cfg, h, best, r, T)


def test_regret_matches_oracle_and_is_nonnegative():
    """Tuners replayed over the same windows: regret_window ≥ 0 everywhere, and for sampled
    tuners both regrets equal the oracle's sum_edp minus the oracle's sweep sums."""
    cfg = named_config("C4")
    T = 6000
    ids = list(range(512))                               # traces 0 and 1, all 256 points
    tb, params, sums, best = _gpu_sweep(cfg, T, [4500, 1500], ids=ids, replay=True)
    reg = tb.regret(sums).cpu().numpy()
    st = tb.stats()
    h = sums.host()
    ok = st["near_tie_steps"] == 0
    assert np.all(reg[:, 0] >= 0.0)
    for i in (0, 15, 100, 255, 256 + 63):
        r = int(params["trace_id"][i])
        acc, _ = oracle.sweep(cfg, r, 0, T)
        ost, _, _ = oracle.run_tuner(cfg, oracle.make_tuner(r, params["alpha0"][i], params["ext_reward_threshold"][i],
                                                            params["hist_k"][i]), T=T)
        if ok[i] and ost["traj_hash"] == int(st["traj_hash"][i]):
            k_off = oracle.offline_arm(acc["S"][:, 2])
            assert reg[i, 0] == st["sum_edp"][i] - acc["O"][0]
            assert reg[i, 1] == st["sum_edp"][i] - acc["S"][k_off, 2]
            assert int(h["koff"][r][5]) == k_off
