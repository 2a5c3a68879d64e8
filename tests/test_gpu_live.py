"""GPU parity of the live two-phase step (agft_select / agft_observe)
against the oracle's live environment, through the C-ABI.

Each window the GPU selects from the tuners' MetricsSnapshot rows; the test then hands it the
pre-drawn measured response (E, TPOT, TTFT) of the arm it chose (agft_inputs.live_inputs — a
seeded table, not a CUDA output).  The oracle replays the same rows and table, following the
GPU's choices under the near-tie rule (ENV.md §4.5); everything else must match as the replay's
parity tests require (trajectory, exact stats and arm counters, A⁻¹ / θ to 1e-9)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from agft_inputs import live_inputs, named_config, tuner_params, with_overrides  # noqa: E402
from paper_2508_01744_b200 import AgftError, TunerBatch  # noqa: E402

from _parity import EXACT_STATS, compare_arms, oracle_tuner  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _live(cfg, n, T, seed, alphas=None):
    cfg = with_overrides(cfg, n_tuners=n, n_traces=n, sweep="none")
    params = tuner_params(cfg)
    if alphas is not None:
        params["alpha0"] = np.asarray(alphas, dtype=np.float64)
    rows, resp = live_inputs(cfg, n, T, seed=seed)
    dev = torch.device("cuda:0")
    rows_d = torch.from_numpy(np.ascontiguousarray(rows.transpose(1, 0, 2)).view(np.int32)).to(dev)   # [T][n][12]
    resp_d = torch.from_numpy(np.ascontiguousarray(resp.transpose(1, 0, 2, 3))).to(dev)               # [T][n][K][3]
    tb = TunerBatch(cfg, params, device=dev)
    chosen = torch.empty((T, n), dtype=torch.int32, device=dev)
    idx = torch.arange(n, device=dev)
    for t in range(T):
        tb.select(rows_d[t], chosen[t])
        tb.observe(resp_d[t][idx, chosen[t].long()].contiguous())
    st = tb.stats()
    torch.cuda.synchronize()
    return cfg, params, rows, resp, tb, chosen.cpu().numpy(), st


def _check(cfg, params, rows, resp, tb, chosen, st, T):
    errs = []
    for i in range(len(params["trace_id"])):
        traj = chosen[:, i].astype(np.uint8)
        ost, oarms, _ = oracle.run_tuner(cfg, oracle_tuner(params, i), T=T, follow=traj,
                                         inject={"rows": rows[i], "resp": resp[i]})
        if ost["follow_violations"]:
            errs.append(f"tuner {i}: {ost['follow_violations']} choices outside the near-tie set")
        if int(st["traj_hash"][i]) != ost["traj_hash"]:
            errs.append(f"tuner {i}: trajectory hash")
        for f in EXACT_STATS:
            if st[f][i] != ost[f]:
                errs.append(f"tuner {i}: stats.{f} {st[f][i]!r} != {ost[f]!r}")
        errs += [f"tuner {i}: {e}" for e in compare_arms(tb.export_arms(i), oarms, cfg["n_arms"])]
    assert not errs, errs[:10]


@pytest.mark.parametrize("name,kw,T", [
    ("C1", {}, 400),                                                # d = 4, 8 arms, no pruning
    ("C2", {}, 700),                                                # full grid, pruning
    ("C2", dict(ph_enable=1, ph_window=20, rf_enable=1), 700),      # + phase switch + refinement
    ("C2", dict(n_arms=40, f_step_mhz=30, hist_min_round=0, hist_min_samples=1), 300),
])
def test_live_parity(name, kw, T):
    cfg = with_overrides(named_config(name), **kw)
    n = 6
    out = _live(cfg, n, T, seed=11, alphas=[0.0, 0.1, 0.5, 1.0, 2.0, 5.0])
    _check(*out, T)
    st = out[-1]
    assert np.all(st["steps"] == T) and np.all(st["base_edp"] == 0.0)
    out[4].close()


def test_live_protocol_errors():
    """Strict select/observe alternation and E_STATE for anything in between."""
    cfg = with_overrides(named_config("C2"), n_tuners=2, n_traces=2)
    params = tuner_params(cfg)
    rows, resp = live_inputs(cfg, 2, 2, seed=3)
    dev = torch.device("cuda:0")
    rows_d = torch.from_numpy(np.ascontiguousarray(rows[:, 0]).view(np.int32)).to(dev)
    resp_d = torch.from_numpy(np.ascontiguousarray(resp[:, 0, 0])).to(dev)
    tb = TunerBatch(cfg, params, device=dev)
    with pytest.raises(AgftError) as e:
        tb.observe(resp_d)
    assert e.value.code == -7
    tb.select(rows_d)
    with pytest.raises(AgftError) as e:
        tb.select(rows_d)
    assert e.value.code == -7
    rec = tb.generate(0, 1)
    with pytest.raises(AgftError) as e:
        tb.replay(rec, 0, 1)
    assert e.value.code == -7
    with pytest.raises(AgftError) as e:
        tb.step(rec)
    assert e.value.code == -7
    tb.observe(resp_d)
    assert tb.t == 1
    rec = tb.generate(1, 3)
    tb.replay(rec, 1, 3)                       # the replay continues from the live state
    assert tb.t == 4
    tb.close()


def test_live_nonfinite_response_freezes_only_that_tuner():
    cfg = with_overrides(named_config("C2"), n_tuners=3, n_traces=3)
    params = tuner_params(cfg)
    rows, resp = live_inputs(cfg, 3, 4, seed=5)
    dev = torch.device("cuda:0")
    tb = TunerBatch(cfg, params, device=dev)
    for t in range(4):
        r = torch.from_numpy(np.ascontiguousarray(rows[:, t]).view(np.int32)).to(dev)
        ch = tb.select(r).cpu().numpy()
        m = resp[np.arange(3), t, np.where(ch < 0, 0, ch)].copy()
        if t == 1:
            m[1, 1] = np.nan
        if t >= 2:
            assert ch[1] == -1                  # AGFT_NEVER: the caller keeps its frequency
        tb.observe(torch.from_numpy(m).to(dev))
    st = tb.stats()
    assert st["flags"][1] & 1 and st["steps"][1] == 1
    assert not (st["flags"][0] & 1) and st["steps"][0] == 4 and st["steps"][2] == 4
    tb.close()
