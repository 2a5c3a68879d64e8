"""Row a6 on the GPU: a constructed exact tie must be flagged by both sides, and the
Eq. 1 scores themselves — not only the trajectories they drive — must match the oracle element by
element (north_star: arm scores to 1e-9 relative).

Tie constructor: at context e1, an arm updated once with
(e1, r) scores r/2 + α/√2 and a fresh arm scores α, equal at α = (r/2)/(1 − 1/√2).  Through the
live API the first reward is 0 (empty window, AMB-3), so: window 0 → arm 0 (fresh tie, lowest k),
r = 0; window 1 → arm 1 (fresh α beats α/√2), EDP = ½·EDP_0 so r = ½; window 2: arm 1 scores
¼ + α/√2 and the fresh arm 2 scores α — tied at α = ¼/(1 − 1/√2) with τ = 1e300 (α_t = α0).
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from agft_inputs import named_config, tuner_params, with_overrides  # noqa: E402
from paper_2508_01744_b200 import TunerBatch  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _e1_rows(n, T):
    """MetricsSnapshot rows whose normalised context is exactly e1: one waiting request
    (x1 = 1 with bounds [0, 1]), every other counter 0 (x2..x7 = 0)."""
    rows = np.zeros((n, T, 12), np.uint32)
    rows[..., 0] = 1
    return rows


@pytest.mark.parametrize("alpha_scale", [1.0, 1.0 + 4e-10, 1.0 - 4e-10, 1.0 + 1e-6])
def test_constructed_tie_is_flagged_on_both_sides(alpha_scale):
    K, d, T = 6, 3, 4
    cfg = with_overrides(named_config("C2"), n_arms=K, d=d, n_tuners=1, n_traces=1, tau=1e300, prune_enable=0)
    alpha = 0.25 / (1.0 - math.sqrt(0.5)) * alpha_scale
    params = tuner_params(cfg)
    params["alpha0"] = np.array([alpha])
    rows = _e1_rows(1, T)
    E0 = 200.0
    resp = np.zeros((1, T, K, 3))
    resp[..., 0] = E0
    resp[..., 1] = 0.02
    resp[0, 1, :, 0] = E0 / 2                      # window 1: EDP halves → r = ½
    resp[..., 2] = 0.1
    tb = TunerBatch(cfg, params, device="cuda:0")
    chosen = []
    for t in range(T):
        ch = tb.select(torch.from_numpy(np.ascontiguousarray(rows[:, t]).view(np.int32)).to("cuda:0"))
        k = ch.cpu().numpy()
        chosen.append(int(k[0]))
        tb.observe(torch.from_numpy(np.ascontiguousarray(resp[np.arange(1), t, k])).to("cuda:0"))
    st = tb.stats()
    ost, _, orec = oracle.run_tuner(cfg, oracle.make_tuner(0, alpha), T=T, follow=np.array(chosen, np.uint8),
                                    record=True, inject={"rows": rows[0], "resp": resp[0]})
    assert chosen[:2] == [0, 1]
    assert ost["follow_violations"] == 0 and int(st["traj_hash"][0]) == ost["traj_hash"]
    # window 2 is the (near-)tie between arm 1 and the fresh arm 2: flagged iff the scores are within
    # 1e-9 relative — on both sides (|α_scale − 1| = 4e-10 still ties, 1e-6 does not)
    tied = abs(alpha_scale - 1.0) < 1e-9
    assert bool(orec["near_tie"][2]) == tied
    assert int(st["near_tie_steps"][0]) == ost["near_tie_steps"] == (1 if tied else 0) + int(orec["near_tie"][3])
    assert chosen[2] in (1, 2)
    tb.close()


def test_scores_element_by_element_across_classes():
    """100 C2 tuners (α swept over 4 decades so the pruning depths differ) replayed on the class
    schedule for 700 windows; then agft_scores at window 700 on the trace's own snapshot row:
    every arm's Eq. 1 score (NaN where pruned) against the oracle's score record of window 700,
    1e-9 relative with a floor of 1e-12 of the tuner's largest |score|."""
    n, T = 100, 700
    cfg = with_overrides(named_config("C2"), n_tuners=n, n_traces=n)
    params = tuner_params(cfg)
    params["alpha0"] = 10.0 ** np.linspace(-2, 1, n)
    params["hist_k"] = np.array([0.5, 1.0, 2.0, 4.0] * (n // 4))
    tb = TunerBatch(cfg, params, device="cuda:0")
    tb.run(T, chunk=350)
    _, raw = tb.generate(T, 1, raw=True)
    g_scores, g_arg = tb.scores(raw[:, 0].contiguous())
    g_scores = g_scores.cpu().numpy()
    g_arg = g_arg.cpu().numpy()
    st = tb.stats()
    worst, checked = 0.0, 0
    for i in range(n):
        tu = oracle.make_tuner(int(params["trace_id"][i]), params["alpha0"][i], params["ext_reward_threshold"][i],
                               params["hist_k"][i])
        ost, _, rec = oracle.run_tuner(cfg, tu, T=T + 1, record=True, scores=True)
        # the GPU's state after T windows is the oracle's state before window T (same trajectory)
        o_st, _, _ = oracle.run_tuner(cfg, tu, T=T)
        assert o_st["traj_hash"] == int(st["traj_hash"][i]), i
        o = rec["scores"][T]
        g = g_scores[i]
        assert np.array_equal(np.isnan(o), np.isnan(g)), i
        live = ~np.isnan(o)
        scale = np.max(np.abs(o[live]))
        err = np.abs(g[live] - o[live])
        assert np.all(err <= 1e-9 * np.abs(o[live]) + 1e-12 * scale), (i, np.max(err))
        worst = max(worst, float(np.max(err / np.maximum(np.abs(o[live]), 1e-300))))
        checked += int(live.sum())
        if not rec["near_tie"][T]:
            assert g_arg[i] == rec["arm"][T], i
    assert checked > n                                  # several arms per tuner still active somewhere
    tb.close()


def test_scores_refused_between_select_and_observe():
    cfg = with_overrides(named_config("C2"), n_tuners=2, n_traces=2)
    tb = TunerBatch(cfg, tuner_params(cfg), device="cuda:0")
    rows = torch.from_numpy(_e1_rows(2, 1)[:, 0].view(np.int32)).to("cuda:0")
    s0, _ = tb.scores(rows)
    assert np.allclose(s0.cpu().numpy(), 1.0)          # fresh arms at e1, t = 0: α0 · 1 = 1
    tb.select(rows)
    import paper_2508_01744_b200 as pkg
    with pytest.raises(pkg.AgftError) as e:
        tb.scores(rows)
    assert e.value.code == -7
    tb.close()
