"""GPU parity of the closed-loop environment ENV-C (ENV.md §6) against
the oracle, through agft_replay_raw: per-tuner and baseline backlogs feed x1, the concurrency
penalty and TTFT, so trajectories, all stats sums (TTFT and the f_max baseline included) and the
arm state must match exactly as in the open-loop parity tests."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from agft_inputs import named_config, tuner_params, with_overrides  # noqa: E402
from paper_2508_01744_b200 import AgftError, TunerBatch  # noqa: E402

from test_gpu_parity import _check, _run  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("kw,T,chunk", [
    (dict(pattern_mode=2), 3000, 700),                          # burst load: backlogs build
    (dict(pattern_mode=2, cl_q_max=12, n_arms=40, f_step_mhz=30), 2000, 4500),
    (dict(pattern_mode=1, ph_enable=1, rf_enable=1), 2500, 1000),  # + phase switch + refinement
    (dict(pattern_mode=2, n_arms=1, prune_enable=0), 1500, 512),   # one low clock: a saturated queue
])
@pytest.mark.parametrize("policy", [0, 1])      # AUTO (SOLO / SEG2 / WIDE classes) and WIDE only
def test_closed_loop_parity(kw, T, chunk, policy):
    cfg = with_overrides(named_config("C2"), cl_enable=1, n_tuners=6, n_traces=6, **kw)
    ids = list(range(6))
    params = tuner_params(cfg, ids)
    params["alpha0"] = np.array([0.0, 0.2, 0.5, 1.0, 2.0, 4.0])
    tb, params, st, traj, gap = _run(cfg, T, params=params, record=ids, chunk=chunk, policy=policy)
    _check(cfg, tb, params, st, ids, T, traj, gap=gap)
    tb.close()


def test_closed_loop_c4_sampled():
    """One C4 trace's 256 hyper-parameter points under ENV-C for 9,000 windows in the bench's
    launch configuration (all classes, SOLO included); a sample checked against the oracle."""
    cfg = with_overrides(named_config("C4"), cl_enable=1, n_traces=1)
    ids = list(range(256))
    params = tuner_params(cfg, ids)
    sample = [0, 15, 48, 63, 100, 200, 255]
    tb, params, st, traj, gap = _run(cfg, 9000, params=params, record=sample, chunk=4500)
    _check(cfg, tb, params, st, sample, 9000, traj, slots={i: s for s, i in enumerate(sample)}, gap=gap)
    tb.close()


def test_closed_loop_changes_the_run_and_open_calls_are_refused():
    base = with_overrides(named_config("C2"), pattern_mode=2, n_tuners=2, n_traces=2, n_arms=1, prune_enable=0)
    T = 1200
    tb_o, _, so, _, _ = _run(base, T)
    tb_c, _, sc, _, _ = _run(with_overrides(base, cl_enable=1), T)
    assert np.all(sc["sum_ttft"] > so["sum_ttft"])           # queued requests wait longer
    assert np.all(sc["base_energy"] >= so["base_energy"])
    rec = tb_c.new_records(1)
    with pytest.raises(AgftError) as e:
        tb_c.replay(rec, T, 1)                                # closed loop needs the raw rows
    assert e.value.code == -1
    with pytest.raises(AgftError):
        tb_c.step(rec)
    tb_o.close()
    tb_c.close()
